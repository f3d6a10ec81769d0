// `offsim` command line: the reference CLI's subcommands (proj/tools/
// offsim_main.cpp:339-411 — simulate, sweep, compare, plan, traffic,
// alloc-plan; same options, outputs and exit codes 0 / 2 validation /
// 3 infeasible / 1 internal) over this repo's drop-in library, plus `run`,
// which executes the configuration on the B200 with the real executor and
// reports the measured iteration next to simulate()'s prediction.
//
// The reference parses arguments with CLI11 (absent here); this is a small
// hand-written parser: one subcommand, positional config path, `--key value`
// options, `--oracle` flag, `--schedules` taking every value up to the next
// option.
#include <chrono>
#include <cmath>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "offsim/executor.hpp"
#include "offsim/json_io.hpp"
#include "offsim/offsim.hpp"

using namespace offsim;

namespace {

struct Args {
  std::string cmd, config;
  std::map<std::string, std::string> opt;
  std::vector<std::string> schedules;
  bool oracle = false;
  bool has(const char* k) const { return opt.count(k) != 0; }
  std::string get(const char* k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
};

const std::map<std::string, std::vector<std::string>> kOptions = {
    {"simulate", {"out", "format", "schedule", "microbatches", "alpha", "split", "emit-plan", "from-plan"}},
    {"sweep", {"out", "format", "m-range", "schedule", "alpha", "split"}},
    {"compare", {"out", "format", "m-range", "split"}},
    {"plan", {"out", "format"}},
    {"traffic", {"out", "format", "schedule", "microbatches", "alpha", "split"}},
    {"alloc-plan", {"count", "size"}},
    {"run", {"out", "format", "schedule", "microbatches", "alpha", "split", "iterations", "warmup", "vocab",
             "nvme-dir", "seed", "device", "lp-bytes", "from-plan", "emit-trace"}},
};

Args parse_args(int argc, char** argv) {
  if (argc < 2) throw ValidationError("usage: offsim <simulate|sweep|compare|plan|traffic|alloc-plan|run> ...");
  Args a;
  a.cmd = argv[1];
  auto known = kOptions.find(a.cmd);
  if (known == kOptions.end()) throw ValidationError("unknown subcommand: " + a.cmd);
  for (int i = 2; i < argc; ++i) {
    std::string t = argv[i];
    if (t.rfind("--", 0) != 0) {
      if (!a.config.empty()) throw ValidationError("unexpected argument: " + t);
      a.config = t;
      continue;
    }
    const std::string key = t.substr(2);
    if (key == "oracle" && a.cmd == "plan") {
      a.oracle = true;
      continue;
    }
    if (key == "schedules" && a.cmd == "compare") {
      while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) a.schedules.push_back(argv[++i]);
      continue;
    }
    bool ok = false;
    for (const auto& k : known->second) ok = ok || k == key;
    if (!ok) throw ValidationError("unknown option --" + key + " for " + a.cmd);
    if (i + 1 >= argc) throw ValidationError("--" + key + " needs a value");
    a.opt[key] = argv[++i];
  }
  if (a.cmd != "alloc-plan" && a.config.empty()) throw ValidationError(a.cmd + ": config file required");
  if (a.has("format") && a.get("format") != "json" && a.get("format") != "csv")
    throw ValidationError("--format must be json or csv");
  return a;
}

int to_int(const std::string& s, const char* what) {
  try {
    size_t n = 0;
    const int v = std::stoi(s, &n);
    if (n != s.size()) throw 0;
    return v;
  } catch (...) {
    throw ValidationError(std::string(what) + " must be an integer");
  }
}
double to_double(const std::string& s, const char* what) {
  try {
    size_t n = 0;
    const double v = std::stod(s, &n);
    if (n != s.size()) throw 0;
    return v;
  } catch (...) {
    throw ValidationError(std::string(what) + " must be a number");
  }
}

ScheduleVariant variant_of(const std::string& s, const char* what) {
  if (s == "vertical") return ScheduleVariant::Vertical;
  if (s == "horizontal") return ScheduleVariant::Horizontal;
  if (s == "single-fb") return ScheduleVariant::SingleFB;
  throw ValidationError(std::string(what) + " must be horizontal|vertical|single-fb");
}

// config file + command-line overrides; a missing split comes from the
// planner's LP (vertical) or is all-SSD (other schedules), as in the reference
RunConfig load(const Args& a, bool fill_split = true) {
  RunConfig cfg = parse_config(a.config);
  if (a.has("schedule")) cfg.schedule.variant = variant_of(a.get("schedule"), "--schedule");
  if (a.has("microbatches")) {
    cfg.num_microbatches = to_int(a.get("microbatches"), "--microbatches");
    if (cfg.num_microbatches < 1) throw ValidationError("--microbatches must be >= 1");
  }
  if (a.has("alpha")) {
    const double al = to_double(a.get("alpha"), "--alpha");
    if (al < 0 || al > 1) throw ValidationError("--alpha must be in [0,1]");
    cfg.schedule.delay_ratio = al;
  }
  if (a.has("split")) {
    std::istringstream in(a.get("split"));
    StorageSplit s;
    char c1 = 0, c2 = 0;
    if (!(in >> s.x_ckpt >> c1 >> s.x_param >> c2 >> s.x_opt) || c1 != ',' || c2 != ',')
      throw ValidationError("--split must be x_ckpt,x_param,x_opt");
    s.validate();
    cfg.split = s;
  }
  if (!cfg.split && fill_split) {
    if (cfg.schedule.variant == ScheduleVariant::Vertical) {
      const PlannerSolution sol = solve_config(cfg.model, cfg.machine, cfg.num_microbatches, cfg.schedule.delay_ratio);
      if (!sol.feasible) throw InfeasibleError("no feasible storage split for this configuration");
      cfg.split = sol.split;
    } else {
      cfg.split = StorageSplit{};
    }
  }
  return cfg;
}

SchedulePlan build(const RunConfig& c) {
  if (c.schedule.variant == ScheduleVariant::Vertical)
    return build_vertical(c.model, c.num_microbatches, *c.split, c.schedule.delay_ratio);
  if (c.schedule.variant == ScheduleVariant::Horizontal) return build_horizontal(c.model, c.num_microbatches, *c.split);
  return build_single_fb(c.model, c.batch, c.schedule.extra_ckpt, *c.split);
}

bool csv(const RunConfig& cfg, const Args& a) {
  return a.has("format") ? a.get("format") == "csv" : cfg.format == OutputFormat::Csv;
}

void emit(const RunConfig& cfg, const Args& a, const std::string& text) {
  const std::string path = a.has("out") ? a.get("out") : cfg.out_path;
  if (path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream out(path);
  if (!out) throw ValidationError("cannot open output path: " + path);
  out << text;
}

std::string kv_csv(const Json& j) {
  std::string s = "key,value\n";
  for (auto it = j.begin(); it != j.end(); ++it)
    if (!it->is_structured()) s += it.key() + "," + it->dump() + "\n";
  return s;
}

std::pair<int, int> m_range(const Args& a) {
  const std::string r = a.get("m-range", "1..8");
  const size_t dots = r.find("..");
  int lo = 0, hi = 0;
  try {
    lo = std::stoi(dots == std::string::npos ? r : r.substr(0, dots));
    hi = dots == std::string::npos ? lo : std::stoi(r.substr(dots + 2));
  } catch (...) {
    throw ValidationError("--m-range must be a..b with integers");
  }
  if (lo < 1 || hi < lo) throw ValidationError("--m-range must satisfy 1 <= a <= b");
  return {lo, hi};
}

std::string fmt(double v) {
  std::ostringstream o;
  o << round_sig(v);
  return o.str();
}

SchedulePlan read_plan(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open plan JSON: " + path);
  Json j;
  try {
    in >> j;
  } catch (const std::exception& e) {
    throw ValidationError(std::string("bad plan JSON: ") + e.what());
  }
  return plan_from_json(j);
}

int cmd_simulate(const Args& a) {
  const RunConfig cfg = load(a);
  SchedulePlan plan;
  if (a.has("from-plan")) {
    plan = read_plan(a.get("from-plan"));
  } else {
    plan = build(cfg);
  }
  if (a.has("emit-plan")) {
    std::ofstream out(a.get("emit-plan"));
    if (!out) throw ValidationError("cannot open --emit-plan path");
    out << plan_to_json(plan).dump(2) << "\n";
  }
  const Json j = report_to_json(simulate(plan, cfg.machine));
  emit(cfg, a, csv(cfg, a) ? kv_csv(j) : j.dump(2) + "\n");
  return 0;
}

int cmd_sweep(const Args& a) {
  if (!a.has("m-range")) throw ValidationError("sweep: --m-range is required");
  const RunConfig cfg = load(a);
  const auto [lo, hi] = m_range(a);
  std::string out = "M,batch,throughput,io_limit,compute_limit,bound_class,note\n";
  for (int m = lo; m <= hi; ++m) {
    RunConfig c = cfg;
    c.num_microbatches = m;
    u64 batch = static_cast<u64>(m) * static_cast<u64>(c.model.microbatch_size);
    if (c.schedule.variant == ScheduleVariant::SingleFB) {
      c.batch = m;
      batch = static_cast<u64>(m);
    }
    const double io = io_roofline(c.model, c.machine, batch, c.split->x_opt);
    const double comp = compute_roofline(c.model, c.machine);
    out += std::to_string(m) + "," + std::to_string(batch) + ",";
    try {
      const SimReport rep = simulate(build(c), c.machine);
      out += fmt(rep.throughput) + "," + fmt(io) + "," + fmt(comp) + "," + rep.bound_class + ",ok\n";
    } catch (const InfeasibleError& e) {
      out += ",," + fmt(comp) + ",infeasible," + e.what() + "\n";
    }
  }
  emit(cfg, a, out);
  return 0;
}

int cmd_compare(const Args& a) {
  if (a.schedules.size() < 2) throw ValidationError("--schedules needs at least two entries");
  const RunConfig base = load(a);
  const auto [lo, hi] = m_range(a);
  std::string out = "schedule";
  for (int m = lo; m <= hi; ++m) out += ",M=" + std::to_string(m);
  out += "\n";
  std::vector<std::vector<double>> rows;
  for (const std::string& tok : a.schedules) {
    RunConfig cfg = base;
    const size_t at = tok.find('@');
    cfg.schedule.variant = variant_of(tok.substr(0, at), "schedule token");
    if (at != std::string::npos) {
      cfg.schedule.delay_ratio = to_double(tok.substr(at + 1), "alpha in schedule token");
      if (cfg.schedule.delay_ratio < 0 || cfg.schedule.delay_ratio > 1)
        throw ValidationError("alpha in schedule token must be in [0,1]");
    }
    out += tok;
    std::vector<double> row;
    for (int m = lo; m <= hi; ++m) {
      RunConfig c = cfg;
      c.num_microbatches = m;
      if (c.schedule.variant == ScheduleVariant::SingleFB) c.batch = m;
      double tp = 0.0;
      try {
        tp = simulate(build(c), c.machine).throughput;
      } catch (const InfeasibleError&) {
      }
      row.push_back(tp);
      out += "," + (tp > 0 ? fmt(tp) : std::string("infeasible"));
    }
    rows.push_back(row);
    out += "\n";
  }
  out += "ratio(last/first)";
  for (size_t i = 0; i < rows.back().size(); ++i)
    out += "," + (rows.front()[i] > 0 && rows.back()[i] > 0 ? fmt(rows.back()[i] / rows.front()[i]) : std::string("n/a"));
  out += "\n";
  emit(base, a, out);
  return 0;
}

int cmd_plan(const Args& a) {
  const RunConfig cfg = load(a, false);
  const PlannerSolution sol = find_optimal_config(cfg.model, cfg.machine);
  if (!sol.feasible)
    throw InfeasibleError(
        "no feasible configuration at any micro-batch count; GPU or CPU memory capacity is the binding constraint");
  Json j = planner_to_json(sol);
  if (a.oracle) {
    const PlannerSolution grid = grid_search_config(cfg.model, cfg.machine, sol.num_microbatches, sol.alpha);
    double dev = 0.0;
    if (grid.feasible) {
      const double x = sol.t_fwd_stage + sol.t_bwd_stage, y = grid.t_fwd_stage + grid.t_bwd_stage;
      dev = std::fabs(x - y) / std::max(y, 1e-300);
    }
    j["oracle_max_deviation"] = round_sig(dev);
  }
  emit(cfg, a, csv(cfg, a) ? kv_csv(j) : j.dump(2) + "\n");
  return 0;
}

int cmd_traffic(const Args& a) {
  const RunConfig cfg = load(a);
  TrafficLedger led;
  if (cfg.schedule.variant == ScheduleVariant::Vertical)
    led = vertical_traffic(cfg.model, cfg.num_microbatches, *cfg.split, cfg.schedule.delay_ratio);
  else if (cfg.schedule.variant == ScheduleVariant::Horizontal)
    led = horizontal_traffic(cfg.model, cfg.num_microbatches, *cfg.split);
  else
    led = single_fb_traffic(cfg.model, cfg.batch, cfg.schedule.extra_ckpt, *cfg.split);
  // JSON unless CSV is asked for (the config default format is JSON)
  const bool json = a.has("format") ? a.get("format") == "json" : cfg.format == OutputFormat::Json;
  emit(cfg, a, json ? ledger_to_json(led).dump(2) + "\n" : ledger_to_csv(led));
  return 0;
}

int cmd_alloc(const Args& a) {
  if (!a.has("count") || !a.has("size")) throw ValidationError("alloc-plan: --count and --size are required");
  u64 size = 0;
  try {
    size = std::stoull(a.get("size"));
  } catch (...) {
    throw ValidationError("--size must be a positive integer (bytes)");
  }
  std::cout << alloc_to_json(plan_alloc(to_int(a.get("count"), "--count"), size)).dump(2) << "\n";
  return 0;
}

// The executed trace in the plan wire format (plan_to_json, the reference's
// `--emit-plan` schema, proj/src/json_io.cpp:142-180) with, per task, one
// record per executed iteration: the resource queue it ran on, its start /
// end (ms from the run start; CUDA events for GPU-side tasks) and the bytes
// physically moved.  Stripping "trace" gives back the input plan.
Json trace_to_json(const SchedulePlan& plan, const std::vector<TraceRecord>& trace) {
  Json j = plan_to_json(plan);
  std::vector<Json> per(plan.tasks.size(), Json::array());
  for (const TraceRecord& r : trace) {
    if (r.task < 0 || r.task >= static_cast<int>(per.size())) throw PlanBugError("trace record of an unknown task");
    per[r.task].push_back(Json{{"iteration", r.iteration},
                               {"resource", resource_name(r.resource)},
                               {"start_ms", r.t_start_ms},
                               {"end_ms", r.t_end_ms},
                               {"physical_bytes", r.physical_bytes}});
  }
  Json& tasks = j["tasks"];
  for (size_t i = 0; i < per.size(); ++i) tasks[i]["trace"] = std::move(per[i]);
  return j;
}

// Executes the configuration on the GPU (bf16 by default; --lp-bytes 4 for
// the fp32 parity mode) with synthetic tokens and random-init weights.
int cmd_run(const Args& a) {
  RunConfig cfg = load(a);
  if (a.has("lp-bytes")) cfg.model.low_precision_bytes = to_int(a.get("lp-bytes"), "--lp-bytes");
  // --from-plan: execute a dumped plan (e.g. the reference CLI's
  // `simulate --emit-plan`) instead of building one from the config
  const SchedulePlan plan = a.has("from-plan") ? read_plan(a.get("from-plan")) : build(cfg);
  ExecConfig ec;
  ec.model = cfg.model;
  ec.vocab_size = a.has("vocab") ? to_int(a.get("vocab"), "--vocab") : 50304;
  ec.nvme_dir = a.get("nvme-dir", "/tmp");
  ec.seed = a.has("seed") ? static_cast<uint64_t>(to_int(a.get("seed"), "--seed")) : 42;
  ec.device = a.has("device") ? to_int(a.get("device"), "--device") : 0;
  const int iters = a.has("iterations") ? to_int(a.get("iterations"), "--iterations") : 3;
  const int warm = a.has("warmup") ? to_int(a.get("warmup"), "--warmup") : 1;
  if (iters < 1 || warm < 0) throw ValidationError("--iterations >= 1 and --warmup >= 0");
  const ModelSpec& m = cfg.model;
  const long long per_it = 1LL * plan.num_microbatches * m.microbatch_size * (m.seq_len + 1);
  std::vector<int32_t> tokens(static_cast<size_t>(per_it) * (iters + warm));
  uint64_t st = ec.seed * 0x9E3779B97F4A7C15ull + 7;
  for (auto& t : tokens) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    t = static_cast<int32_t>((st >> 33) % static_cast<uint64_t>(ec.vocab_size));
  }
  ec.record_trace = a.has("emit-trace");
  Executor ex(plan, ec);
  if (warm > 0) ex.run(warm, tokens.data());
  const ExecReport rep = ex.run(iters, tokens.data() + static_cast<size_t>(per_it) * warm);
  const double it_s = rep.total_ms / 1e3 / iters;
  const SimReport sim = simulate(plan, cfg.machine);
  Json j;
  j["iterations"] = iters;
  j["measured_iteration_time"] = round_sig(it_s);
  j["measured_throughput"] = round_sig(plan.num_microbatches * m.microbatch_size * cfg.machine.num_gpus / it_s);
  j["tokens_per_s"] = round_sig(1.0 * plan.num_microbatches * m.microbatch_size * m.seq_len / it_s);
  j["simulated_iteration_time"] = round_sig(sim.iteration_time);
  j["ledger_equals_plan"] = rep.ledger.bytes == plan_traffic(plan).bytes;
  Json losses = Json::array();
  for (double l : rep.losses) losses.push_back(round_sig(l));
  j["losses"] = losses;
  j["traffic"] = ledger_to_json(rep.ledger);
  j["extension_traffic"] = ledger_to_json(rep.extension);
  if (a.has("emit-trace")) {
    std::ofstream out(a.get("emit-trace"));
    if (!out) throw ValidationError("cannot open --emit-trace path");
    out << trace_to_json(plan, rep.trace).dump() << "\n";
  }
  emit(cfg, a, csv(cfg, a) ? kv_csv(j) : j.dump(2) + "\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    if (a.cmd == "simulate") return cmd_simulate(a);
    if (a.cmd == "sweep") return cmd_sweep(a);
    if (a.cmd == "compare") return cmd_compare(a);
    if (a.cmd == "plan") return cmd_plan(a);
    if (a.cmd == "traffic") return cmd_traffic(a);
    if (a.cmd == "alloc-plan") return cmd_alloc(a);
    return cmd_run(a);
  } catch (const ValidationError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const InfeasibleError& e) {
    std::cerr << "infeasible: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 1;
  }
}
