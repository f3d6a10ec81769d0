// Configuration planner (reference API: proj/include/offsim/planner.hpp;
// the paper's Algorithm 1, restated from proj/src/planner.cpp:49-256).
//
// One pipeline stage of the vertical schedule (one layer, all M micro-
// batches) occupies six resources; its time is the largest occupancy.  Every
// occupancy is an affine function of the CPU-resident fractions
// x = (x_ckpt, x_param, x_opt) — SSD bytes shrink linearly as more is kept
// in DRAM — so "stage time = max of affine terms" is linear-programmable:
// t_f >= term_k(x) for every forward term, t_b likewise, minimise
// t_f + t_b.  The same term list evaluates the exact stage times of a split
// (solve_config's report, grid_search_config), so LP and evaluation cannot
// drift apart.
//
// Terms per layer (bytes: p params bf16, c checkpoint per MB, o optimizer
// state, g fp32 grads; shard_* per-GPU PCIe shards; dp the DP degree):
//   fwd: GPU M t_f | CPU a P / thr | H2D (shard_p + (M-1) c) | D2H M c |
//        SSD read  (1-a)(1-x_p) p + a (1-x_o) o
//        SSD write (1-x_c) M c dp + a ((1-x_o) o + (1-x_p) p)
//   bwd: GPU M t_b | CPU (1-a) P / thr | H2D (shard_p + (2M-1) c) |
//        D2H (shard_g + (M-1) c) |
//        SSD read  (1-x_p) p + (1-x_c) M c dp + (1-a)(1-x_o) o
//        SSD write (1-a) ((1-x_o) o + (1-x_p) p)
// A full-duplex SSD contributes separate read and write terms, a half-duplex
// one their sum.  Constraints: x <= 1; DRAM holds grads, double buffers and
// the resident fractions; the delayed slice's grads fit in memory reclaimed
// from consumed params / checkpoints (the builder's check, schedule.cpp:
// 293-305); GPU residency is split-independent.
#include <algorithm>
#include <array>
#include <cmath>

#include "offsim/offsim.hpp"

namespace offsim {

namespace {

// value(x) = k + w . x  (seconds)
struct Affine {
  double k = 0.0;
  std::array<double, 3> w{0.0, 0.0, 0.0};
  double at(const StorageSplit& x) const { return k + w[0] * x.x_ckpt + w[1] * x.x_param + w[2] * x.x_opt; }
};
Affine constant(double v) { return Affine{v, {0.0, 0.0, 0.0}}; }
// bytes = base - sum(drop_i * x_i); time = bytes / bw
Affine bytes_over(double base, std::array<double, 3> drop, double bw) {
  return Affine{base / bw, {-drop[0] / bw, -drop[1] / bw, -drop[2] / bw}};
}
Affine sum(const Affine& a, const Affine& b) {
  return Affine{a.k + b.k, {a.w[0] + b.w[0], a.w[1] + b.w[1], a.w[2] + b.w[2]}};
}

struct Stage {
  std::vector<Affine> fwd, bwd;
  double resident_const = 0.0;             // DRAM bytes independent of x
  std::array<double, 3> resident{0, 0, 0};  // DRAM bytes per unit of x
  double alpha_grads = 0.0;                 // delayed-slice grads to park
  std::array<double, 3> reclaim{0, 0, 0};   // DRAM reclaimable per unit of x
  double gpu_need = 0.0;
  double N = 0.0, M = 0.0;

  static double worst(const std::vector<Affine>& terms, const StorageSplit& x) {
    double t = 0.0;
    for (const Affine& a : terms) t = std::max(t, a.at(x));
    return t;
  }
};

Stage build_stage(const ModelSpec& model, const MachineSpec& mc, int big_m, double a) {
  const LayerSizes ls = derive_layer_sizes(model);
  const double p = static_cast<double>(ls.param_bytes_low), c = static_cast<double>(ls.ckpt_bytes_per_mb);
  const double o = static_cast<double>(ls.opt_state_bytes), g = static_cast<double>(ls.grad_bytes_full);
  const double sp = static_cast<double>(chunk_size(ls.param_bytes_low, model.data_parallel_degree, 0));
  const double sg = static_cast<double>(chunk_size(ls.grad_bytes_full, model.data_parallel_degree, 0));
  const double P = static_cast<double>(ls.param_elements);
  const double M = big_m, N = model.num_layers, dp = model.data_parallel_degree;
  Stage s;
  s.N = N;
  s.M = M;
  // forward stage
  s.fwd.push_back(constant(M * mc.fwd_compute_time_per_layer_per_mb));
  s.fwd.push_back(constant(a * P / mc.cpu_step_throughput));
  s.fwd.push_back(constant((sp + (M - 1) * c) / mc.pcie_h2d_bw));
  s.fwd.push_back(constant(M * c / mc.pcie_d2h_bw));
  const Affine rf = bytes_over((1 - a) * p + a * o, {0.0, (1 - a) * p, a * o}, mc.ssd_read_bw);
  const Affine wf = bytes_over(M * c * dp + a * (o + p), {M * c * dp, a * p, a * o}, mc.ssd_write_bw);
  // backward stage
  s.bwd.push_back(constant(M * mc.bwd_compute_time_per_layer_per_mb));
  s.bwd.push_back(constant((1 - a) * P / mc.cpu_step_throughput));
  s.bwd.push_back(constant((sp + (2 * M - 1) * c) / mc.pcie_h2d_bw));
  s.bwd.push_back(constant((sg + (M - 1) * c) / mc.pcie_d2h_bw));
  const Affine rb = bytes_over(p + M * c * dp + (1 - a) * o, {M * c * dp, p, (1 - a) * o}, mc.ssd_read_bw);
  const Affine wb = bytes_over((1 - a) * (o + p), {0.0, (1 - a) * p, (1 - a) * o}, mc.ssd_write_bw);
  if (mc.ssd_duplex) {
    s.fwd.insert(s.fwd.end(), {rf, wf});
    s.bwd.insert(s.bwd.end(), {rb, wb});
  } else {
    s.fwd.push_back(sum(rf, wf));
    s.bwd.push_back(sum(rb, wb));
  }
  // DRAM: all grads, double-buffered ckpt / param / opt working sets, and
  // the resident fractions of every layer
  s.resident_const = N * g + 2 * M * c * dp + 2 * p + 2 * o;
  s.resident = {M * c * N * dp, p * N, o * N};
  s.alpha_grads = a * N * g;
  s.reclaim = {M * N * c, a * N * p, 0.0};
  s.gpu_need = 2 * sp + 2 * sg + 4 * c + static_cast<double>(mc.gpu_working_set_bytes);
  return s;
}

void finish(PlannerSolution& sol, const Stage& st, const ModelSpec& model, const MachineSpec& mc) {
  sol.t_fwd_stage = Stage::worst(st.fwd, sol.split);
  sol.t_bwd_stage = Stage::worst(st.bwd, sol.split);
  sol.iteration_estimate = st.N * (sol.t_fwd_stage + sol.t_bwd_stage) + mc.fixed_overhead_time;
  sol.throughput_estimate =
      st.M * static_cast<double>(model.microbatch_size) * static_cast<double>(mc.num_gpus) / sol.iteration_estimate;
  sol.feasible = true;
}

void check_args(const ModelSpec& model, const MachineSpec& mc, int big_m, double alpha) {
  model.validate();
  mc.validate();
  if (big_m < 1) throw ValidationError("num_microbatches must be >= 1");
  if (!(alpha >= 0.0 && alpha <= 1.0)) throw ValidationError("delay ratio alpha must be in [0,1]");
}

}  // namespace

PlannerSolution solve_config(const ModelSpec& model, const MachineSpec& mc, int big_m, double alpha) {
  check_args(model, mc, big_m, alpha);
  PlannerSolution sol;
  sol.num_microbatches = big_m;
  sol.alpha = alpha;
  const Stage st = build_stage(model, mc, big_m, alpha);
  if (st.gpu_need > static_cast<double>(mc.gpu_mem_bytes)) return sol;

  // variables: x_ckpt, x_param, x_opt, t_fwd, t_bwd
  constexpr int kTf = 3, kTb = 4, kVars = 5;
  std::vector<std::vector<double>> A;
  std::vector<double> b;
  for (int i = 0; i < 3; ++i) {  // x_i <= 1
    std::vector<double> r(kVars, 0.0);
    r[static_cast<size_t>(i)] = 1.0;
    A.push_back(r);
    b.push_back(1.0);
  }
  auto stage_rows = [&](const std::vector<Affine>& terms, int t) {  // term(x) <= t
    for (const Affine& a : terms) {
      std::vector<double> r(kVars, 0.0);
      for (int i = 0; i < 3; ++i) r[static_cast<size_t>(i)] = a.w[static_cast<size_t>(i)];
      r[static_cast<size_t>(t)] = -1.0;
      A.push_back(r);
      b.push_back(-a.k);
    }
  };
  stage_rows(st.fwd, kTf);
  stage_rows(st.bwd, kTb);
  {  // DRAM capacity
    std::vector<double> r(kVars, 0.0);
    for (int i = 0; i < 3; ++i) r[static_cast<size_t>(i)] = st.resident[static_cast<size_t>(i)];
    A.push_back(r);
    b.push_back(static_cast<double>(mc.cpu_usable_dram_bytes) - st.resident_const);
  }
  {  // delayed-slice residency; a relative margin keeps the split clear of the
     // builder's integer-rounded check
    std::vector<double> r(kVars, 0.0);
    for (int i = 0; i < 3; ++i) r[static_cast<size_t>(i)] = -st.reclaim[static_cast<size_t>(i)];
    A.push_back(r);
    b.push_back(-st.alpha_grads * (1.0 + 1e-6));
  }
  // objective: stage times, minus a small reward for every byte kept off
  // the SSD (so equal-time splits prefer DRAM), with a lexicographic nudge
  // opt > params > checkpoints for exact ties
  const double offloadable = st.resident[0] + st.resident[1] + st.resident[2];
  const double lambda = 1.0 / (1e6 * offloadable);
  std::vector<double> c(kVars, 0.0);
  c[0] = -lambda * st.resident[0] - 1e-10;
  c[1] = -lambda * st.resident[1] - 2e-10;
  c[2] = -lambda * st.resident[2] - 3e-10;
  c[kTf] = 1.0;
  c[kTb] = 1.0;
  const LpResult lp = solve_lp(A, b, c);
  if (!lp.feasible || !lp.bounded) return sol;
  sol.split.x_ckpt = std::clamp(lp.x[0], 0.0, 1.0);
  sol.split.x_param = std::clamp(lp.x[1], 0.0, 1.0);
  sol.split.x_opt = std::clamp(lp.x[2], 0.0, 1.0);
  finish(sol, st, model, mc);
  return sol;
}

PlannerSolution find_optimal_config(const ModelSpec& model, const MachineSpec& mc) {
  // M = 1, 2, ...: best alpha on the grid {0.01, ..., 0.50} per M; stop at the
  // first M that does not beat the incumbent by more than 1%
  PlannerSolution best;
  for (int m = 1; m <= 1024; ++m) {
    // best alpha of this M; throughputs equal to 1e-12 relative are ties
    // (last-bit LP noise), resolved toward the smaller alpha
    PlannerSolution here;
    for (int k = 1; k <= 50; ++k) {
      const PlannerSolution s = solve_config(model, mc, m, k / 100.0);
      if (s.feasible && (!here.feasible || s.throughput_estimate > here.throughput_estimate * (1.0 + 1e-12))) here = s;
    }
    if (!here.feasible) break;
    if (best.feasible && here.throughput_estimate <= 1.01 * best.throughput_estimate) break;
    best = here;
  }
  return best;
}

PlannerSolution grid_search_config(const ModelSpec& model, const MachineSpec& mc, int big_m, double alpha,
                                   int steps) {
  check_args(model, mc, big_m, alpha);
  if (steps < 1) throw ValidationError("grid steps must be >= 1");
  PlannerSolution best;
  best.num_microbatches = big_m;
  best.alpha = alpha;
  const Stage st = build_stage(model, mc, big_m, alpha);
  if (st.gpu_need > static_cast<double>(mc.gpu_mem_bytes)) return best;
  const double dram = static_cast<double>(mc.cpu_usable_dram_bytes);
  double best_t = 0.0;
  for (int ic = 0; ic <= steps; ++ic)
    for (int ip = 0; ip <= steps; ++ip)
      for (int io = 0; io <= steps; ++io) {
        StorageSplit x;
        x.x_ckpt = static_cast<double>(ic) / steps;
        x.x_param = static_cast<double>(ip) / steps;
        x.x_opt = static_cast<double>(io) / steps;
        const std::array<double, 3> xv{x.x_ckpt, x.x_param, x.x_opt};
        double mem = st.resident_const, rec = 0.0;
        for (int i = 0; i < 3; ++i) {
          mem += st.resident[static_cast<size_t>(i)] * xv[static_cast<size_t>(i)];
          rec += st.reclaim[static_cast<size_t>(i)] * xv[static_cast<size_t>(i)];
        }
        if (mem > dram || st.alpha_grads > rec + 1e-9) continue;
        const double t = Stage::worst(st.fwd, x) + Stage::worst(st.bwd, x);
        if (!best.feasible || t < best_t) {
          best.feasible = true;
          best_t = t;
          best.split = x;
        }
      }
  if (best.feasible) finish(best, st, model, mc);
  return best;
}

double whole_model_projection(const PlannerSolution& sol, const ModelSpec& model, const MachineSpec& mc) {
  return static_cast<double>(model.num_layers) * (sol.t_fwd_stage + sol.t_bwd_stage) + mc.fixed_overhead_time;
}

}  // namespace offsim
