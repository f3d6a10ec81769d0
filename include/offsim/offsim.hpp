// offsim — drop-in plan/ledger/engine API of the GreedySnake B200 framework.
//
// This single header carries every declaration of the `offsim::` namespace that
// the reference exposes under proj/include/offsim/*.hpp for the hot path
// (vertical schedule + alpha-delayed optimizer step).  The per-topic headers
// (offsim/schedule.hpp, offsim/traffic.hpp, ...) forward here so that code
// written against the reference includes compile unchanged.
//
// Reference interfaces mirrored (file:line under /root/reference/proj):
//   errors + byte rounding     include/offsim/types.hpp:13-60
//   ModelSpec / LayerSizes     include/offsim/model.hpp:11-49
//   MachineSpec / LinkKind     include/offsim/machine.hpp:8-38
//   plan IR + builders         include/offsim/schedule.hpp:12-86
//   TrafficLedger + ledgers    include/offsim/traffic.hpp:14-50
//   simulate / SimReport       include/offsim/simulator.hpp:11-34
//   rooflines                  include/offsim/roofline.hpp:12-17
// The real executor that replaces simulate() on B200 is declared in
// offsim/executor.hpp.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace offsim {

using u64 = std::uint64_t;

// ---------------------------------------------------------------- errors
// Exit-code convention of the reference CLI: Validation -> 2, Infeasible -> 3,
// PlanBug -> 1 (proj/tools/offsim_main.cpp:400-409).
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};
struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& what) : std::runtime_error(what) {}
};
struct PlanBugError : std::logic_error {
  explicit PlanBugError(const std::string& what) : std::logic_error(what) {}
};

// ------------------------------------------------------- byte rounding
// The builders and the closed-form ledgers must round identically; every
// fractional split of a byte count goes through these four helpers.
inline u64 scaled_portion(u64 bytes, double fraction) {
  if (!(fraction > 0.0)) return 0;
  if (fraction >= 1.0) return bytes;
  const auto r = static_cast<u64>(std::llround(fraction * static_cast<double>(bytes)));
  return r < bytes ? r : bytes;
}
inline u64 cpu_portion(u64 bytes, double cpu_fraction) { return scaled_portion(bytes, cpu_fraction); }
inline u64 ssd_portion(u64 bytes, double cpu_fraction) { return bytes - cpu_portion(bytes, cpu_fraction); }
// Piece `index` of `total` cut into `parts` near-equal pieces; the first
// total % parts pieces carry one extra byte so the pieces sum to `total`.
inline u64 chunk_size(u64 total, int parts, int index) {
  const u64 n = static_cast<u64>(parts);
  return total / n + (static_cast<u64>(index) < total % n ? 1u : 0u);
}

// ------------------------------------------------------------- geometry
struct ModelSpec {
  int num_layers = 1;       // N
  int hidden_dim = 1;       // h
  int num_heads = 1;
  int seq_len = 1;          // s
  int microbatch_size = 1;  // b
  int low_precision_bytes = 2;   // parameter / activation storage width
  int full_precision_bytes = 4;  // gradient / optimizer-state width
  int optimizer_states_per_element = 3;  // master, m, v
  int data_parallel_degree = 1;
  void validate() const;
};

// One transformer layer carries exactly 12*h^2 parameters (QKV 3h^2, out-proj
// h^2, FC1 4h^2, FC2 4h^2; bias-free linears, non-affine LayerNorm).
struct LayerSizes {
  u64 param_elements = 0;
  u64 param_bytes_low = 0;
  u64 grad_bytes_full = 0;
  u64 opt_state_bytes = 0;
  u64 ckpt_elements_per_mb = 0;  // b*s*h
  u64 ckpt_bytes_per_mb = 0;
};
struct ModelTotals {
  u64 param_elements = 0;
  u64 param_bytes_low = 0;
  u64 ckpt_bytes_per_mb = 0;
  u64 opt_state_bytes = 0;
  u64 grad_bytes_full = 0;
};
LayerSizes derive_layer_sizes(const ModelSpec& spec);
ModelTotals model_totals(const ModelSpec& spec);

// -------------------------------------------------------------- machine
enum class LinkKind { PCIe_H2D, PCIe_D2H, SSD_Read, SSD_Write };

struct MachineSpec {
  u64 gpu_mem_bytes = 0;
  u64 cpu_usable_dram_bytes = 0;
  double pcie_h2d_bw = 0;   // bytes/s
  double pcie_d2h_bw = 0;
  double ssd_read_bw = 0;
  double ssd_write_bw = 0;
  double fwd_compute_time_per_layer_per_mb = 0;  // s
  double bwd_compute_time_per_layer_per_mb = 0;  // s, recompute included
  double cpu_step_throughput = 0;                // elements/s
  double fixed_overhead_time = 0;                // s per iteration
  int num_gpus = 1;
  u64 gpu_working_set_bytes = 0;
  bool ssd_duplex = true;
  void validate() const;
};
double transfer_time(u64 bytes, LinkKind link, const MachineSpec& machine);
double optimizer_step_time(u64 elements, const MachineSpec& machine);
const char* link_name(LinkKind link);

// ------------------------------------------------------------- plan IR
enum class ScheduleVariant { SingleFB, Horizontal, Vertical };
struct ScheduleKind {
  ScheduleVariant variant = ScheduleVariant::Vertical;
  bool extra_ckpt = false;
  double delay_ratio = 0.0;  // alpha
};
// CPU-resident fractions; the rest of each kind lives on SSD.  Gradients are
// always CPU-resident.
struct StorageSplit {
  double x_ckpt = 0.0;
  double x_param = 0.0;
  double x_opt = 0.0;
  void validate() const;
};
enum class TaskKind { FwdCompute, RecomputeAndBwd, CpuStep, Xfer, FixedOps };
enum class DataKind { Param, Ckpt, GradAccum, InterlayerGrad, OptState };
constexpr int kAllMicrobatches = -1;

struct Task {
  int id = 0;
  TaskKind kind = TaskKind::Xfer;
  int layer = -1;
  int microbatch = kAllMicrobatches;
  int stage = 0;
  DataKind data = DataKind::Param;     // Xfer only
  LinkKind link = LinkKind::PCIe_H2D;  // Xfer only
  u64 bytes = 0;                       // Xfer only, > 0
  u64 elements = 0;                    // CpuStep only
  std::vector<int> deps;               // ids < id, sorted, unique
  int cross_iter_dep = -1;             // id in the previous iteration, or -1
};

struct SchedulePlan {
  ScheduleKind kind;
  int num_microbatches = 1;
  int num_layers = 1;
  StorageSplit split;
  std::vector<Task> tasks;
  u64 samples_per_iteration = 0;  // per GPU
  double compute_scale = 1.0;
  u64 gpu_static_bytes = 0;
  u64 cpu_peak_bytes = 0;
  std::string gpu_binding;
};

SchedulePlan build_horizontal(const ModelSpec& model, int num_microbatches,
                              const StorageSplit& split);
SchedulePlan build_vertical(const ModelSpec& model, int num_microbatches,
                            const StorageSplit& split, double alpha);
SchedulePlan build_single_fb(const ModelSpec& model, int batch, bool extra_ckpt,
                             const StorageSplit& split);
long long overlap_window(const SchedulePlan& plan);

// -------------------------------------------------------------- ledgers
// bytes[link][data] per iteration.
struct TrafficLedger {
  static constexpr int kLinks = 4;
  static constexpr int kData = 5;
  std::array<std::array<u64, kData>, kLinks> bytes{};

  u64& at(LinkKind l, DataKind d) { return bytes[static_cast<size_t>(l)][static_cast<size_t>(d)]; }
  u64 at(LinkKind l, DataKind d) const { return bytes[static_cast<size_t>(l)][static_cast<size_t>(d)]; }
  u64 link_total(LinkKind l) const {
    u64 s = 0;
    for (u64 v : bytes[static_cast<size_t>(l)]) s += v;
    return s;
  }
  u64 total() const {
    u64 s = 0;
    for (int l = 0; l < kLinks; ++l) s += link_total(static_cast<LinkKind>(l));
    return s;
  }
  bool operator==(const TrafficLedger&) const = default;
};
const char* data_name(DataKind d);
TrafficLedger horizontal_traffic(const ModelSpec& model, int num_microbatches,
                                 const StorageSplit& split);
TrafficLedger vertical_traffic(const ModelSpec& model, int num_microbatches,
                               const StorageSplit& split, double alpha);
TrafficLedger single_fb_traffic(const ModelSpec& model, int batch, bool extra_ckpt,
                                const StorageSplit& split);
TrafficLedger plan_traffic(const SchedulePlan& plan);

// ------------------------------------------------------------ simulator
enum class Resource { GPU, CPU, H2D, D2H, SSD_R, SSD_W };
inline constexpr int kNumResources = 6;
const char* resource_name(Resource r);

struct SimReport {
  double iteration_time = 0.0;
  double throughput = 0.0;  // samples/s over all GPUs
  TrafficLedger ledger;
  u64 gpu_mem_needed = 0;
  u64 cpu_mem_needed = 0;
  std::map<std::string, double> utilization;
  std::string bound_class;
};
SimReport simulate(const SchedulePlan& plan, const MachineSpec& machine);

// Which in-order resource queue a task occupies (simulator.cpp:24-43 of the
// reference); the executor uses the same mapping for its queues.
Resource task_resource(const Task& t, bool ssd_duplex);
// Structural checks every consumer of a plan may rely on (ids, topological
// deps, cross-iteration range).  Throws PlanBugError.
void check_plan(const SchedulePlan& plan);

// ------------------------------------------------------------- roofline
double io_roofline(const ModelSpec& model, const MachineSpec& machine, u64 batch_samples,
                   double x_opt = 0.0);
double compute_roofline(const ModelSpec& model, const MachineSpec& machine);

// -------------------------------------------------------------- simplex
// (reference API: proj/include/offsim/simplex.hpp)
struct LpResult {
  bool feasible = false;
  bool bounded = true;
  std::vector<double> x;
  double objective = 0.0;
};
// min c.x  s.t.  A x <= b, x >= 0 (dense two-phase primal simplex, Bland's rule).
LpResult solve_lp(const std::vector<std::vector<double>>& A, const std::vector<double>& b,
                  const std::vector<double>& c);

// -------------------------------------------------------------- planner
// (reference API: proj/include/offsim/planner.hpp; Algorithm 1 of the paper)
struct PlannerSolution {
  bool feasible = false;
  int num_microbatches = 0;
  double alpha = 0.0;
  StorageSplit split;
  double t_fwd_stage = 0.0;  // per layer, all micro-batches
  double t_bwd_stage = 0.0;
  double iteration_estimate = 0.0;
  double throughput_estimate = 0.0;  // samples/s over all GPUs
};
PlannerSolution solve_config(const ModelSpec& model, const MachineSpec& machine, int num_microbatches,
                             double alpha);
PlannerSolution find_optimal_config(const ModelSpec& model, const MachineSpec& machine);
PlannerSolution grid_search_config(const ModelSpec& model, const MachineSpec& machine, int num_microbatches,
                                   double alpha, int steps = 100);
double whole_model_projection(const PlannerSolution& sol, const ModelSpec& model, const MachineSpec& machine);

// ---------------------------------------------------------------- alloc
// (reference API: proj/include/offsim/alloc.hpp) grouping of equal pinned
// buffers into power-of-two requests
struct AllocRequest {
  int buffer_count = 0;
  u64 requested_bytes = 0;
  u64 granted_bytes = 0;
};
struct AllocPlan {
  std::vector<AllocRequest> requests;
  u64 total_requested = 0;
  u64 total_granted = 0;
};
u64 next_pow2(u64 v);
AllocPlan plan_alloc(int count, u64 buffer_bytes);

// --------------------------------------------------------------- config
// (reference API: proj/include/offsim/config.hpp) INI run description with
// sections [model], [machine], optional [schedule] / [output].
enum class OutputFormat { Json, Csv };
struct RunConfig {
  ModelSpec model;
  MachineSpec machine;
  ScheduleKind schedule;
  int num_microbatches = 1;
  int batch = 1;                      // SingleFB only
  std::optional<StorageSplit> split;  // planner fills it when absent
  OutputFormat format = OutputFormat::Json;
  std::string out_path;               // empty = stdout
};
RunConfig parse_config(const std::string& path);

}  // namespace offsim
