// TEST INFRASTRUCTURE ONLY (oracle): a C-ABI shim over the reference's own
// offsim library, compiled from the sources under /root/reference/proj by
// oracle/Makefile into oracle/_ref/liboffsim_ref.so.  Only tests/ and
// bench.py's reference/cpu_baseline legs may load it.  It exposes the
// reference builders, ledgers and simulator so parity tests can diff this
// repo's drop-in library against the reference byte for byte.
#include <cstdlib>
#include <cstring>
#include <string>

#include "offsim/json_io.hpp"
#include "offsim/planner.hpp"
#include "offsim/roofline.hpp"
#include "offsim/simplex.hpp"
#include "offsim/schedule.hpp"
#include "offsim/simulator.hpp"
#include "offsim/traffic.hpp"

using namespace offsim;

namespace {
thread_local std::string g_err;

ModelSpec model_of(const int* m) {
  ModelSpec s;
  s.num_layers = m[0]; s.hidden_dim = m[1]; s.num_heads = m[2]; s.seq_len = m[3];
  s.microbatch_size = m[4]; s.low_precision_bytes = m[5]; s.full_precision_bytes = m[6];
  s.optimizer_states_per_element = m[7]; s.data_parallel_degree = m[8];
  return s;
}
StorageSplit split_of(const double* x) {
  StorageSplit s; s.x_ckpt = x[0]; s.x_param = x[1]; s.x_opt = x[2]; return s;
}
MachineSpec machine_of(const double* d) {
  MachineSpec mc;
  mc.gpu_mem_bytes = static_cast<u64>(d[0]); mc.cpu_usable_dram_bytes = static_cast<u64>(d[1]);
  mc.pcie_h2d_bw = d[2]; mc.pcie_d2h_bw = d[3]; mc.ssd_read_bw = d[4]; mc.ssd_write_bw = d[5];
  mc.fwd_compute_time_per_layer_per_mb = d[6]; mc.bwd_compute_time_per_layer_per_mb = d[7];
  mc.cpu_step_throughput = d[8]; mc.fixed_overhead_time = d[9]; mc.num_gpus = static_cast<int>(d[10]);
  mc.gpu_working_set_bytes = static_cast<u64>(d[11]); mc.ssd_duplex = d[12] != 0.0;
  return mc;
}
char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
template <typename F> int guard(F&& f) {
  try { f(); return 0; }
  catch (const ValidationError& e) { g_err = e.what(); return 2; }
  catch (const InfeasibleError& e) { g_err = e.what(); return 3; }
  catch (const std::exception& e) { g_err = e.what(); return 1; }
}
SchedulePlan build(int variant, const int* m, int mbs, int extra, const double* x, double alpha) {
  if (variant == 2) return build_vertical(model_of(m), mbs, split_of(x), alpha);
  if (variant == 1) return build_horizontal(model_of(m), mbs, split_of(x));
  return build_single_fb(model_of(m), mbs, extra != 0, split_of(x));
}
}  // namespace

extern "C" {
const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }
// variant: 0 single-fb, 1 horizontal, 2 vertical.  *out = plan_to_json(...).dump()
int ref_plan_json(int variant, const int* model, int mbs, int extra, const double* split,
                  double alpha, char** out) {
  return guard([&] { *out = dup(plan_to_json(build(variant, model, mbs, extra, split, alpha)).dump()); });
}
// Closed-form ledger, out[link*5 + data].
int ref_ledger(int variant, const int* model, int mbs, int extra, const double* split, double alpha,
               unsigned long long* out) {
  return guard([&] {
    TrafficLedger t;
    if (variant == 2) t = vertical_traffic(model_of(model), mbs, split_of(split), alpha);
    else if (variant == 1) t = horizontal_traffic(model_of(model), mbs, split_of(split));
    else t = single_fb_traffic(model_of(model), mbs, extra != 0, split_of(split));
    for (int l = 0; l < 4; ++l)
      for (int d = 0; d < 5; ++d) out[l * 5 + d] = t.bytes[l][d];
  });
}
// Planner: mode 0 solve_config(M, alpha), 1 find_optimal_config, 2
// grid_search_config(M, alpha, steps).  out = {feasible, M, alpha, x_ckpt,
// x_param, x_opt, t_fwd, t_bwd, iteration, throughput}
int ref_planner(int mode, const int* model, const double* machine, int mbs, double alpha, int steps, double* out) {
  return guard([&] {
    PlannerSolution s = mode == 0   ? solve_config(model_of(model), machine_of(machine), mbs, alpha)
                        : mode == 1 ? find_optimal_config(model_of(model), machine_of(machine))
                                    : grid_search_config(model_of(model), machine_of(machine), mbs, alpha, steps);
    const double v[10] = {s.feasible ? 1.0 : 0.0, (double)s.num_microbatches, s.alpha, s.split.x_ckpt,
                          s.split.x_param, s.split.x_opt, s.t_fwd_stage, s.t_bwd_stage, s.iteration_estimate,
                          s.throughput_estimate};
    std::memcpy(out, v, sizeof(v));
  });
}
// out = {io_roofline(model, machine, batch, x_opt), compute_roofline(model, machine)}  (roofline.cpp:8-33)
int ref_rooflines(const int* model, const double* machine, unsigned long long batch, double x_opt, double* out) {
  return guard([&] {
    out[0] = io_roofline(model_of(model), machine_of(machine), batch, x_opt);
    out[1] = compute_roofline(model_of(model), machine_of(machine));
  });
}
// solve_lp over a dense row-major A [m x n]: out = {feasible, bounded, objective, x...}
int ref_solve_lp(int m, int n, const double* A, const double* b, const double* c, double* out) {
  return guard([&] {
    std::vector<std::vector<double>> a(static_cast<size_t>(m), std::vector<double>(static_cast<size_t>(n)));
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) a[i][j] = A[i * n + j];
    LpResult r = solve_lp(a, std::vector<double>(b, b + m), std::vector<double>(c, c + n));
    out[0] = r.feasible; out[1] = r.bounded; out[2] = r.objective;
    for (int j = 0; j < n && j < (int)r.x.size(); ++j) out[3 + j] = r.x[j];
  });
}
// report_to_json(simulate(plan_from_json(plan), machine)).dump()
int ref_simulate_json(const char* plan_json, const double* machine, char** out) {
  return guard([&] {
    SchedulePlan p = plan_from_json(Json::parse(plan_json));
    *out = dup(report_to_json(simulate(p, machine_of(machine))).dump());
  });
}
}
