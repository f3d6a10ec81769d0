// The B200 executor: runs a SchedulePlan for real.
//
// This is the slot the reference fills with its discrete-event model
// (`SimReport simulate(const SchedulePlan&, const MachineSpec&)`,
// proj/include/offsim/simulator.hpp:34).  Every plan task is executed on the
// resource simulate() would charge it to, in the same per-resource order
// (proj/src/simulator.cpp:117-122):
//
//   GPU    FwdCompute / RecomputeAndBwd / FixedOps -> compute CUDA stream
//   H2D    Xfer PCIe_H2D                           -> copy stream (pinned DRAM -> HBM)
//   D2H    Xfer PCIe_D2H                           -> copy stream (HBM -> pinned DRAM)
//   CPU    CpuStep                                 -> host cores (OptTier::Host), or the
//                                                     optimizer stream: fused Adam on the GPU,
//                                                     state in HBM or streamed through it
//   SSD_R  Xfer SSD_Read                           -> NVMe file reads (O_DIRECT, thread pool)
//   SSD_W  Xfer SSD_Write                          -> NVMe file writes
//
// Cross-resource dependencies become CUDA events / host completions; the
// plan's cross_iter_dep edges chain consecutive iterations, so the alpha
// slice of iteration i's optimizer step overlaps iteration i+1's forward.
// The trace (task, resource, start, end, bytes) of every executed task sums
// to plan_traffic(plan) exactly; transfers the GPU optimizer adds on top of
// the reference model are reported in a separate extension ledger.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "offsim/offsim.hpp"

namespace offsim {

// Where the plan's CPU-resident optimizer fraction (split.x_opt) lives and
// which processor runs CpuStep on it.  SSD-resident bytes always round-trip
// through the NVMe file and a pinned staging slot.
enum class OptTier {
  Auto = 0,    // HBM when it fits (< 60% of free HBM), else Stream
  Hbm = 1,     // kept in HBM (B200: 180 GB); fused Adam kernel in place
  Stream = 2,  // pinned DRAM, streamed through HBM per step (upload -> fused Adam -> download pipeline)
  Host = 3,    // pinned DRAM, stepped by the host cores where it lives: the reference's CpuStep
               // (simulator.cpp:24-43), gradients from the plan's GradAccum D2H, no extra PCIe bytes
};

struct AdamConfig {
  float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.0f;
};

struct ExecConfig {
  ModelSpec model;          // geometry; low_precision_bytes 2 = bf16, 4 = fp32 parity mode
  int vocab_size = 50304;   // embedding / tied LM head (FixedOps), off the ledger
  AdamConfig adam;
  uint64_t seed = 42;       // weight init (N(0,0.02), out-proj / sqrt(2N))
  int device = 0;
  std::string nvme_dir = "/tmp";  // directory of the NVMe tier file
  bool odirect = true;
  OptTier opt_tier = OptTier::Auto;
  bool record_trace = false;   // per-task timestamps (adds event records)
  bool profile_kernels = false;  // CUDA-event timing per kernel class on the compute stream
  // ZeRO-3 data parallelism: one executor per rank, model.data_parallel_degree
  // == world; the job's 128-byte communicator id (rank 0 draws it with
  // gs_comm_unique_id, the launcher broadcasts it) names the one-node
  // peer-memory rendezvous (engine/peer_comm.hpp).
  int rank = 0, world = 1;
  std::vector<uint8_t> comm_id;
  bool force_collectives = false;  // run the sharded code path even at world == 1 (tests)
  // SSD-resident bytes have no permanent DRAM copy: each data kind stages
  // them through a ring of this many per-layer pinned slots (slot = layer %
  // ring); reuse of a slot is ordered by the executor's hazard edges.
  int ssd_ring_layers = 8;
  int host_threads = 0;  // OptTier::Host worker threads (0: (hardware threads - 4) / world, at least 1)
};

struct TraceRecord {
  int iteration;
  int task;
  Resource resource;
  double t_start_ms, t_end_ms;  // relative to the run start (GPU tasks: CUDA events)
  u64 bytes;                    // logical bytes (the plan's)
  u64 physical_bytes;           // bytes actually moved (NVMe rounds to 4 KiB)
  double t_host_ms = 0.0;       // host time the dispatcher began enqueueing it (dependencies dispatched)
};

struct ExecReport {
  // measured, per iteration
  std::vector<double> losses;
  std::vector<double> iteration_ms;   // end-to-end time of each iteration (GPU clock)
  double total_ms = 0.0;              // whole run, CUDA events
  TrafficLedger ledger;               // logical bytes moved in the LAST iteration (== plan_traffic)
  TrafficLedger extension;            // GPU-optimizer traffic outside the reference model
  TrafficLedger physical;             // bytes physically moved in the last iteration
  u64 gpu_bytes_allocated = 0;
  u64 host_pinned_bytes = 0;
  int gpu_launches = 0;               // kernels launched by the run (all iterations)
  std::vector<TraceRecord> trace;     // when record_trace
};

class Executor {
 public:
  // Builds device / host / NVMe state for `plan` (weights initialised from
  // cfg.seed; optimizer state zero).  Throws ValidationError / InfeasibleError.
  Executor(const SchedulePlan& plan, const ExecConfig& cfg);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  // Runs `iterations` chained iterations of the plan.  tokens: host (or
  // device, if tokens_on_device) int32 [iterations][M][b][s+1].
  ExecReport run(int iterations, const int32_t* tokens, bool tokens_on_device = false);
  // Applies the pending alpha slice of the last iteration's step and the
  // pending embedding step ("flush"); idempotent.
  void flush();
  // fp32 master weights: layers [N][12h^2], fixed [(V+s)*h] (wte then wpe).
  void read_params(float* layers, float* fixed);
  // fp32 optimizer moments, same layout as read_params (fixed_m / fixed_v:
  // the embedding / position table's, [(V+s)*h]; may be null).
  void read_moments(float* layer_m, float* layer_v, float* fixed_m = nullptr, float* fixed_v = nullptr);
  // Per kernel class of the last run (profile_kernels): algorithmic flops,
  // summed CUDA-event milliseconds and launches.  Classes: gemm,
  // attention_fwd, attention_bwd, layernorm, other.
  struct KernelTotals {
    double flops[5];       // sampled launches
    double ms[5];          // sampled launches
    int launches[5];       // sampled launches
    long long total[5];    // all launches of the class
    // tcgen05 GEMM launches sampled by in-kernel %globaltimer span (first
    // CTA start .. last CTA exit), not bracketed by events
    double span_flops = 0, span_ms = 0;
    int span_launches = 0;
  };
  KernelTotals kernel_profile() const;
  // 0 disables per-kernel timing; n times one launch in n per class.
  void set_profiling(int stride);
  // Per-task trace for the following runs (timing events are created on
  // first use).
  void set_trace(bool on);

  const SchedulePlan& plan() const;
  const ExecConfig& config() const;

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

// One-call form mirroring simulate(plan, machine).
ExecReport execute(const SchedulePlan& plan, const ExecConfig& cfg, int iterations,
                   const int32_t* tokens);

}  // namespace offsim
