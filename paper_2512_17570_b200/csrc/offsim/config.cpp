// INI run descriptions (reference API: proj/include/offsim/config.hpp,
// parse_config; schema, defaults and error messages follow
// proj/src/config.cpp:124-225 so configs and their diagnostics carry over).
//
// Implementation: the file is tokenised into section -> key -> raw value,
// then every section is checked against a table of field descriptors (name,
// type, required/default, store) instead of hand-written per-field code; the
// same table rejects unknown keys.
#include <cctype>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <vector>

#include "offsim/offsim.hpp"

namespace offsim {

namespace {

using Section = std::map<std::string, std::string>;

std::string strip(const std::string& s) {
  size_t a = 0, z = s.size();
  while (a < z && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
  while (z > a && std::isspace(static_cast<unsigned char>(s[z - 1]))) --z;
  return s.substr(a, z - a);
}

std::map<std::string, Section> read_ini(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open config file: " + path);
  std::map<std::string, Section> ini;
  std::string line, current;
  for (int no = 1; std::getline(in, line); ++no) {
    const std::string t = strip(line);
    if (t.empty() || t[0] == '#' || t[0] == ';') continue;
    if (t.size() >= 2 && t.front() == '[' && t.back() == ']') {
      current = strip(t.substr(1, t.size() - 2));
      ini[current];
      continue;
    }
    const size_t eq = t.find('=');
    const std::string where = path + ":" + std::to_string(no) + ": ";
    if (eq == std::string::npos) throw ValidationError(where + "expected key = value");
    if (current.empty()) throw ValidationError(where + "key before any [section]");
    ini[current][strip(t.substr(0, eq))] = strip(t.substr(eq + 1));
  }
  return ini;
}

enum class Kind { Integer, Number, Boolean, Text };

struct Field {
  const char* key;
  Kind kind;
  bool required;
  std::function<void(const std::string&)> store;  // raw value (validated by kind)
};

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Integer: return "integer";
    case Kind::Number: return "number";
    case Kind::Boolean: return "boolean (true/false)";
    case Kind::Text: return "string";
  }
  return "value";
}

template <typename T>
T convert(const std::string& section, const Field& f, const std::string& raw) {
  std::istringstream in(raw);
  T v{};
  in >> v;
  std::string extra;
  if (!in || (in >> extra, !extra.empty()))
    throw ValidationError("field " + section + "." + f.key + " must be a " + kind_name(f.kind) + ", got '" + raw + "'");
  return v;
}

bool convert_bool(const std::string& section, const Field& f, const std::string& raw) {
  if (raw == "true" || raw == "1") return true;
  if (raw == "false" || raw == "0") return false;
  throw ValidationError("field " + section + "." + f.key + " must be a " + kind_name(f.kind) + ", got '" + raw + "'");
}

// Applies `fields` to `sec`: unknown keys and missing required keys throw.
void apply(const std::string& name, const Section& sec, const std::vector<Field>& fields) {
  for (const auto& kv : sec) {
    bool known = false;
    for (const Field& f : fields) known = known || kv.first == f.key;
    if (!known) throw ValidationError("unknown field " + name + "." + kv.first);
  }
  for (const Field& f : fields) {
    auto it = sec.find(f.key);
    if (it == sec.end()) {
      if (f.required) throw ValidationError("missing required field " + name + "." + f.key);
      continue;
    }
    f.store(it->second);
  }
}

void unit_interval(double v, const char* field) {
  if (v < 0.0 || v > 1.0) throw ValidationError(std::string("field ") + field + " must be in [0,1]");
}

}  // namespace

RunConfig parse_config(const std::string& path) {
  auto ini = read_ini(path);
  for (const char* s : {"model", "machine"})
    if (!ini.count(s)) throw ValidationError(std::string("missing [") + s + "] section");
  RunConfig cfg;

  auto I = [](const char* sec, const char* key, bool req, auto set) {
    Field f{key, Kind::Integer, req, nullptr};
    f.store = [f, sec, set](const std::string& raw) { set(convert<long long>(sec, f, raw)); };
    return f;
  };
  auto R = [](const char* sec, const char* key, bool req, auto set) {
    Field f{key, Kind::Number, req, nullptr};
    f.store = [f, sec, set](const std::string& raw) { set(convert<double>(sec, f, raw)); };
    return f;
  };
  auto B = [](const char* sec, const char* key, auto set) {
    Field f{key, Kind::Boolean, false, nullptr};
    f.store = [f, sec, set](const std::string& raw) { set(convert_bool(sec, f, raw)); };
    return f;
  };
  auto T = [](const char* key, auto set) {
    Field f{key, Kind::Text, false, nullptr};
    f.store = [set](const std::string& raw) { set(raw); };
    return f;
  };

  ModelSpec& m = cfg.model;  // defaults (lp 2, fp 4, 3 states, dp 1) from ModelSpec
  apply("model", ini["model"],
        {I("model", "num_layers", true, [&](long long v) { m.num_layers = static_cast<int>(v); }),
         I("model", "hidden_dim", true, [&](long long v) { m.hidden_dim = static_cast<int>(v); }),
         I("model", "num_heads", true, [&](long long v) { m.num_heads = static_cast<int>(v); }),
         I("model", "seq_len", true, [&](long long v) { m.seq_len = static_cast<int>(v); }),
         I("model", "microbatch_size", true, [&](long long v) { m.microbatch_size = static_cast<int>(v); }),
         I("model", "low_precision_bytes", false, [&](long long v) { m.low_precision_bytes = static_cast<int>(v); }),
         I("model", "full_precision_bytes", false, [&](long long v) { m.full_precision_bytes = static_cast<int>(v); }),
         I("model", "optimizer_states_per_element", false,
           [&](long long v) { m.optimizer_states_per_element = static_cast<int>(v); }),
         I("model", "data_parallel_degree", false,
           [&](long long v) { m.data_parallel_degree = static_cast<int>(v); })});
  m.validate();

  MachineSpec& mc = cfg.machine;
  mc.num_gpus = 1;
  mc.fixed_overhead_time = 0.0;
  mc.gpu_working_set_bytes = 0;
  mc.ssd_duplex = true;
  apply("machine", ini["machine"],
        {I("machine", "gpu_mem_bytes", true, [&](long long v) { mc.gpu_mem_bytes = static_cast<u64>(v); }),
         I("machine", "cpu_usable_dram_bytes", true, [&](long long v) { mc.cpu_usable_dram_bytes = static_cast<u64>(v); }),
         R("machine", "pcie_h2d_bw", true, [&](double v) { mc.pcie_h2d_bw = v; }),
         R("machine", "pcie_d2h_bw", true, [&](double v) { mc.pcie_d2h_bw = v; }),
         R("machine", "ssd_read_bw", true, [&](double v) { mc.ssd_read_bw = v; }),
         R("machine", "ssd_write_bw", true, [&](double v) { mc.ssd_write_bw = v; }),
         R("machine", "fwd_compute_time_per_layer_per_mb", true,
           [&](double v) { mc.fwd_compute_time_per_layer_per_mb = v; }),
         R("machine", "bwd_compute_time_per_layer_per_mb", true,
           [&](double v) { mc.bwd_compute_time_per_layer_per_mb = v; }),
         R("machine", "cpu_step_throughput", true, [&](double v) { mc.cpu_step_throughput = v; }),
         R("machine", "fixed_overhead_time", false, [&](double v) { mc.fixed_overhead_time = v; }),
         I("machine", "num_gpus", false, [&](long long v) { mc.num_gpus = static_cast<int>(v); }),
         I("machine", "gpu_working_set_bytes", false, [&](long long v) { mc.gpu_working_set_bytes = static_cast<u64>(v); }),
         B("machine", "ssd_duplex", [&](bool v) { mc.ssd_duplex = v; })});
  mc.validate();

  if (ini.count("schedule")) {
    std::string variant = "vertical";
    long long mbs = 1, batch = 1;
    double alpha = 0.0;
    bool extra = false, any_split = false;
    StorageSplit sp;
    apply("schedule", ini["schedule"],
          {T("variant", [&](const std::string& v) { variant = v; }),
           I("schedule", "microbatches", false, [&](long long v) { mbs = v; }),
           R("schedule", "alpha", false, [&](double v) { alpha = v; }),
           I("schedule", "batch", false, [&](long long v) { batch = v; }),
           B("schedule", "extra_ckpt", [&](bool v) { extra = v; }),
           R("schedule", "x_ckpt", false, [&](double v) { sp.x_ckpt = v, any_split = true; }),
           R("schedule", "x_param", false, [&](double v) { sp.x_param = v, any_split = true; }),
           R("schedule", "x_opt", false, [&](double v) { sp.x_opt = v, any_split = true; })});
    if (variant == "vertical") cfg.schedule.variant = ScheduleVariant::Vertical;
    else if (variant == "horizontal") cfg.schedule.variant = ScheduleVariant::Horizontal;
    else if (variant == "single-fb") cfg.schedule.variant = ScheduleVariant::SingleFB;
    else
      throw ValidationError("field schedule.variant must be one of horizontal|vertical|single-fb, got '" + variant +
                            "'");
    if (mbs < 1) throw ValidationError("field schedule.microbatches must be >= 1");
    unit_interval(alpha, "schedule.alpha");
    cfg.num_microbatches = static_cast<int>(mbs);
    cfg.schedule.delay_ratio = alpha;
    cfg.batch = static_cast<int>(batch);
    cfg.schedule.extra_ckpt = extra;
    if (any_split) {
      unit_interval(sp.x_ckpt, "schedule.x_ckpt");
      unit_interval(sp.x_param, "schedule.x_param");
      unit_interval(sp.x_opt, "schedule.x_opt");
      cfg.split = sp;
    }
  }
  if (ini.count("output")) {
    std::string fmt = "json";
    apply("output", ini["output"], {T("format", [&](const std::string& v) { fmt = v; }),
                                    T("path", [&](const std::string& v) { cfg.out_path = v; })});
    if (fmt == "json") cfg.format = OutputFormat::Json;
    else if (fmt == "csv") cfg.format = OutputFormat::Csv;
    else throw ValidationError("field output.format must be json or csv, got '" + fmt + "'");
  }
  return cfg;
}

}  // namespace offsim
