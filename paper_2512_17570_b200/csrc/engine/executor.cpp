// The B200 executor (offsim/executor.hpp): runs a vertical (snake) or
// horizontal plan with real kernels, real PCIe DMA and real NVMe I/O.
//
// Structure
//  * One dispatcher thread per plan resource (GPU, CPU, H2D, D2H, SSD_R,
//    SSD_W), each walking its tasks in plan order, iteration after iteration
//    (the in-order discipline of proj/src/simulator.cpp:108-126).
//  * Stream-backed resources record a CUDA event per task instance; a
//    dependency on another stream task is a cudaStreamWaitEvent, on a host
//    task a host wait.  cross_iter_dep edges bind to the previous iteration.
//  * Buffer reuse hazards the plan leaves implicit (parity-indexed HBM
//    staging slots, the gradient ring, NVMe read staging) are derived once by
//    a WAR/WAW pass over two unrolled iterations and added as extra edges
//    pointing backwards in (iteration, plan id) order, so no deadlock is
//    possible.
//  * Each data kind lives in a "blob" cut into segments by the split's byte
//    boundaries (types.hpp:35-53 rounding) and by the immediate/delayed
//    element boundary.  DRAM segments are pinned images.  SSD segments live
//    only in a 4 KiB-aligned region of the NVMe file (the authoritative
//    copy); they pass through a pinned staging slot drawn from a per-kind
//    ring of cfg.ssd_ring_layers layers (slot = layer % ring), which the
//    plan's SSD reads fill and its SSD writes drain.  DRAM use is therefore
//    independent of the SSD-resident bytes, and every SSD byte the plan
//    names really round-trips through the file.
#include "offsim/executor.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <thread>

#include "host_adam.hpp"
#include "host_tiers.hpp"
#include "kernels.h"
#include "layer_ops.hpp"
#include "peer_comm.hpp"

namespace offsim {

using gs::DType;
using namespace gs::engine;

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}


// ------------------------------------------------------------ weight init
// Bit-identical to oracle/gs_oracle.c (gso_splitmix64 / gso_normal /
// gso_init_layer / gso_init_fixed).
uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
double normal_at(uint64_t key, uint64_t i) {
  const uint64_t a = splitmix64(key + 2 * i), b = splitmix64(key + 2 * i + 1);
  const double u1 = static_cast<double>((a >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}
uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream + 0x632BE59BD9B4E019ull));
}
template <typename F>
void parallel_for(long long n, F&& f) {
  const int nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < (1 << 16) || nt == 1) {
    f(0LL, n);
    return;
  }
  std::vector<std::thread> ts;
  const long long per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const long long lo = t * per, hi = std::min(n, lo + per);
    if (lo < hi) ts.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

uint16_t f32_to_bf16(float f) {  // round to nearest even (finite inputs)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}

// ------------------------------------------------------------ tiers
enum class Tier { Dram, Ssd, Hbm };
struct Segment {
  u64 lo = 0, hi = 0;  // logical byte range within the blob
  Tier tier = Tier::Dram;
  uint8_t* img = nullptr;  // Dram: pinned image; Ssd: the layer's staging-ring slot
  uint8_t* rd = nullptr;   // Ssd: same staging slot (NVMe reads land here)
  uint8_t* dev = nullptr;  // HBM (Hbm)
  u64 file_off = 0;        // NVMe region (Ssd)
  u64 size() const { return hi - lo; }
};
struct Blob {
  u64 size = 0;
  std::vector<Segment> segs;
};

// Source selection for an upload of a blob range.
enum class Src { Image, ReadStaging, Auto };

// ------------------------------------------------------------ hazards
struct ExtraDep {
  int task;
  int offset;  // 0 = same iteration, -1 = previous
};

}  // namespace

// =========================================================================
struct Executor::Impl {
  SchedulePlan plan;
  ExecConfig cfg;
  Dims d;
  int N = 0, M = 0;
  u64 P = 0, pb = 0, cb = 0;
  u64 el_now = 0, el_late = 0;
  bool horizontal = false;
  int grad_ring = 3;
  // ZeRO-3 data parallelism: rank R of W owns elements
  // [e_lo, e_hi) of every layer (shards of Ps = ceil(P / W), the last one
  // padded); params are all-gathered per stage, gradients reduce-scattered.
  int W = 1, R = 0;
  u64 Ps = 0, e_lo = 0, e_hi = 0, n_my = 0, loc_now = 0, loc_late = 0;
  bool dp = false;
  std::vector<float*> grad_shard;  // [ring] reduce-scatter output (aliases grad_slot when !dp)
  // Collectives over peer memory (engine/peer_comm.hpp).  Parameter
  // all-gather, pipelined per H2D chunk: each landed chunk of this rank's
  // shard is announced (kParamReady) on s_h2d, and s_ag copies the peers'
  // same chunk out of their HBM into the gathered layer buffer.  Gradient
  // reduce-scatter after a layer's last backward micro-batch on s_rs (off
  // the compute stream: it overlaps the next stage).  Counters are running
  // sequence numbers identical on every rank (same plan, same order).
  std::unique_ptr<PeerComm> peer;
  int pb_param[2] = {-1, -1}, pb_fx_grad = -1, pb_fx_red = -1;
  std::vector<int> pb_grad;
  cudaStream_t s_ag = nullptr, s_rs = nullptr;
  cudaEvent_t ev_ag[2] = {nullptr, nullptr}, ev_h2d_chunk = nullptr, ev_bwd_done = nullptr;
  std::vector<cudaEvent_t> ev_rs;   // [grad_ring] shard of slot k reduced
  uint32_t param_q = 0, grad_q = 0, fixed_q = 0;
  uint32_t param_last[2] = {0, 0};  // last chunk sequence gathered into dev_param[p]
  std::vector<uint32_t> grad_last;  // [grad_ring] last reduce-scatter sequence that read slot k
  float* fx_red = nullptr;          // this rank's shard of the summed embedding gradient
  long long fx_shard = 0;           // ceil(n_fixed / W)
  void fixed_allreduce(cudaStream_t st);

  // streams
  cudaStream_t s_gpu = nullptr, s_h2d = nullptr, s_d2h = nullptr, s_opt = nullptr;

  // device state
  std::vector<void*> dev_allocs;
  u64 dev_bytes = 0;
  void* dev_param[2] = {nullptr, nullptr};
  std::vector<float*> grad_slot;
  std::vector<float*> retain;  // [N] el_late floats
  float *fx_master = nullptr, *fx_m = nullptr, *fx_v = nullptr, *fx_grad = nullptr;
  void* fx_lp = nullptr;
  long long n_fixed = 0;
  Workspace ws;
  KernelProfiler prof;
  std::vector<void*> in_x, out_y, in_g, out_g;  // [2*M] each, index p*M+m
  int32_t* dev_tok[2] = {nullptr, nullptr};
  double* dev_loss = nullptr;  // [loss_cap] per run iteration
  int* dev_bad_tokens = nullptr;  // count of out-of-vocabulary token ids seen by the run
  int loss_cap = 0;
  // Optimizer-state streaming (state not resident in HBM): a ring of
  // staging slots, each one chunk of [master, m, v] (12 B/element) plus its
  // low-precision output.  Chunk c's upload (s_opt_up), fused Adam (s_opt)
  // and download (s_opt_dn) run as a three-stage pipeline, so the H2D and
  // D2H directions and the kernel overlap each other and the plan's own
  // transfers on s_h2d / s_d2h.
  static constexpr int kOptRing = 4;
  struct OptSlot {
    float* state = nullptr;
    void* lp = nullptr;
    cudaEvent_t up = nullptr, comp = nullptr, free_ = nullptr;
    bool used = false;
  };
  std::array<OptSlot, kOptRing> oring;
  int oring_next = 0;
  cudaStream_t s_opt_up = nullptr, s_opt_dn = nullptr;
  cudaEvent_t ev_opt_begin = nullptr, ev_opt_end = nullptr;
  long long chunk = 0;

  // host state
  PinnedArena arena;
  std::unique_ptr<NvmeFile> nvme;
  int ring_k = 1;                                     // staging slots per kind
  std::vector<uint8_t*> ring_param, ring_opt, ring_ckpt;  // [ring_k] ([ring_k * M] for ckpt)
  bool ssd_param = false, ssd_opt = false, ssd_ckpt = false;
  std::vector<Blob> param_blob, opt_blob;  // [N]
  std::vector<Blob> ckpt_blob;             // [N*M]
  std::vector<uint8_t*> host_grad;         // [host_grad_ring], slot = layer % ring
  int host_grad_ring = 1;
  // OptTier::Host: CpuStep runs on the host cores (the reference's resource
  // model).  The GradAccum D2H lands the immediate slice of the layer's
  // gradient in host_grad (ring) and the alpha-delayed slice in
  // host_retain[layer], which the next iteration's forward-phase step reads.
  bool host_step = false;
  std::vector<float*> host_retain;  // [N] loc_late floats
  std::unique_ptr<ThreadPool> host_pool;
  std::vector<uint8_t*> host_ilg;          // [2*M]
  int32_t* tok_pinned = nullptr;
  long long tok_capacity = 0;

  // task bookkeeping
  std::vector<Resource> res_of;
  std::vector<std::vector<int>> queue;  // per resource, task ids in plan order
  std::vector<std::vector<ExtraDep>> extra;
  std::vector<char> is_stream;          // task completes via CUDA event
  std::vector<char> fwd_phase;          // emitted before the first RecomputeAndBwd
  std::vector<u64> chunk_lo;            // param H2D: byte offset of the chunk
  std::vector<std::array<cudaEvent_t, 3>> ev_done;
  std::vector<std::array<cudaEvent_t, 3>> ev_start;  // trace mode
  std::vector<std::atomic<int>> done_iter;
  std::mutex mu;
  std::condition_variable cv;
  std::array<std::atomic<int>, kNumResources> finished{};
  std::atomic<bool> failed{false};
  std::string error;

  // run state
  long long global_iter = 0;  // iterations completed before this run
  long long fixed_done = 0;   // embedding grads of iterations < fixed_done are applied
  // per layer: global iteration whose alpha-slice grads are retained / applied
  std::unique_ptr<std::atomic<long long>[]> late_ready, late_applied;
  const int32_t* run_tokens = nullptr;
  bool run_tokens_dev = false;
  std::atomic<int> launches{0};
  // ledgers (last iteration)
  TrafficLedger led_logical, led_ext, led_phys;
  std::mutex led_mu;
  int last_iter = -1;
  std::vector<TraceRecord> trace;
  std::mutex trace_mu;
  // GS_HOST_PROF=1: host seconds the GPU dispatcher spends waiting on
  // dependencies vs enqueueing kernels (printed to stderr after each run)
  bool host_prof = false;
  double host_wait_s = 0.0, host_enqueue_s = 0.0;
  std::chrono::steady_clock::time_point host_base;
  cudaEvent_t ev_base = nullptr;

  // ------------------------------------------------------------ setup
  Impl(const SchedulePlan& p, const ExecConfig& c);
  ~Impl();
  void* dmalloc(u64 bytes);
  // ssd: byte ranges [lo, hi) of the blob that live on the NVMe file; the
  // rest is CPU-resident (pinned DRAM, or HBM when hbm_for_cpu)
  Blob make_blob(u64 size, const std::vector<std::pair<u64, u64>>& ssd, bool hbm_for_cpu,
                 std::vector<uint8_t*>& ring, int slot);
  void init_weights();
  void build_tasks();
  void hazards();

  // ------------------------------------------------------------ data movement
  u64 upload(const Blob& b, u64 lo, u64 hi, void* dst, Src src, cudaStream_t st, u64 delayed_lo);
  u64 download(Blob& b, u64 lo, u64 hi, const void* src, cudaStream_t st);
  u64 ssd_io(Blob& b, u64 lo, u64 hi, bool write);

  // ------------------------------------------------------------ execution
  void dispatch(Resource r, int iterations);
  void wait_dep(int dep, int iter, bool on_stream, cudaStream_t st);
  void run_task(int t, int it);
  void compute_task(const Task& t, int it);
  void step_task(const Task& t, int it);
  void xfer_task(const Task& t, int it, u64& phys);
  cudaStream_t stream_of(Resource r) const;
  int first_mb(int st) const { return st % 2 == 0 ? 0 : M - 1; }
  int last_mb(int st) const { return st % 2 == 0 ? M - 1 : 0; }
  // forward-phase optimizer work (CpuStep, OptState I/O, Param SSD write) is
  // the delayed alpha slice of the previous iteration's step
  bool delayed(const Task& t) const { return fwd_phase[static_cast<size_t>(t.id)] != 0; }
  // src: where SSD-resident state is read from — the NVMe read staging for
  // plan steps (a plan SSD read precedes each), the image for flush().
  // OptTier::Host: the same step on the host cores, in place on the state's
  // pinned images (DRAM segments, or the NVMe staging slot the plan's
  // OptState SSD read filled); grad is a host pointer.
  void apply_adam_host(int layer, u64 e0, u64 e1, const float* grad, int step);
  void apply_adam(int layer, u64 e0, u64 e1, const float* grad, int step, cudaStream_t st, int it,
                  Src src = Src::ReadStaging);
  void note_ledger(int it, const Task& t, u64 phys);
  void note_ext(int it, LinkKind l, DataKind dk, u64 bytes);
};

// =========================================================================
Executor::Impl::Impl(const SchedulePlan& p, const ExecConfig& c) : plan(p), cfg(c) {
  check_plan(plan);
  const ModelSpec& ms = cfg.model;
  ms.validate();
  if (plan.kind.variant == ScheduleVariant::SingleFB)
    throw ValidationError("executor: single-fb plans are outside the hot path");
  horizontal = plan.kind.variant == ScheduleVariant::Horizontal;
  if (ms.low_precision_bytes != 2 && ms.low_precision_bytes != 4)
    throw ValidationError("executor: low_precision_bytes must be 2 (bf16) or 4 (fp32)");
  if (ms.full_precision_bytes != 4 || ms.optimizer_states_per_element != 3)
    throw ValidationError("executor: fp32 gradients and three Adam states required");
  if (ms.hidden_dim % ms.num_heads || ms.hidden_dim / ms.num_heads > 128 || ms.hidden_dim > 12288)
    throw ValidationError("executor: head_dim must divide hidden and be <= 128; hidden <= 12288");
  if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world)
    throw ValidationError("executor: rank must be in [0, world)");
  if (ms.data_parallel_degree != cfg.world)
    throw ValidationError("executor: model.data_parallel_degree must equal the number of ranks (world)");
  if (cfg.world > 1 && horizontal)
    throw ValidationError("executor: data-parallel execution covers the vertical schedule");
  if (plan.num_layers != ms.num_layers) throw ValidationError("executor: plan and model disagree on num_layers");
  if (cfg.vocab_size < 2) throw ValidationError("executor: vocab_size must be >= 2");
  if (cfg.world > 1 && (12ull * ms.hidden_dim * ms.hidden_dim) % static_cast<u64>(cfg.world) != 0)
    throw ValidationError("executor: 12*hidden^2 must divide by the number of ranks (equal ZeRO-3 shards)");
  {
    // Buffers are sized from cfg.model, transfers from the plan's task bytes:
    // the plan must be the one the builder produces for this model (a plan
    // built for another width / dp degree / precision would overrun them).
    // A reference-dumped plan passes: the builders are byte-identical.
    const SchedulePlan want = horizontal ? build_horizontal(ms, plan.num_microbatches, plan.split)
                                         : build_vertical(ms, plan.num_microbatches, plan.split, plan.kind.delay_ratio);
    if (want.tasks.size() != plan.tasks.size())
      throw ValidationError("executor: plan does not match the model (" + std::to_string(plan.tasks.size()) +
                            " tasks, the model's plan has " + std::to_string(want.tasks.size()) + ")");
    for (size_t i = 0; i < want.tasks.size(); ++i) {
      const Task &a = plan.tasks[i], &b = want.tasks[i];
      if (a.kind != b.kind || a.layer != b.layer || a.microbatch != b.microbatch || a.stage != b.stage ||
          a.data != b.data || a.link != b.link || a.bytes != b.bytes || a.elements != b.elements ||
          a.deps != b.deps || a.cross_iter_dep != b.cross_iter_dep)
        throw ValidationError("executor: plan task " + std::to_string(i) +
                              " does not match the model's plan (bytes / geometry / dp degree differ)");
    }
  }

  N = ms.num_layers;
  M = plan.num_microbatches;
  d.b = ms.microbatch_size;
  d.s = ms.seq_len;
  d.h = ms.hidden_dim;
  d.H = ms.num_heads;
  d.V = cfg.vocab_size;
  d.dt = ms.low_precision_bytes == 2 ? DType::BF16 : DType::F32;
  const LayerSizes ls = derive_layer_sizes(ms);
  P = ls.param_elements;
  pb = ls.param_bytes_low;
  cb = ls.ckpt_bytes_per_mb;
  el_late = horizontal ? 0 : scaled_portion(P, plan.kind.delay_ratio);
  el_now = P - el_late;
  W = cfg.world;
  R = cfg.rank;
  dp = W > 1 || cfg.force_collectives;
  Ps = (P + static_cast<u64>(W) - 1) / static_cast<u64>(W);
  e_lo = std::min<u64>(P, static_cast<u64>(R) * Ps);
  e_hi = std::min<u64>(P, e_lo + Ps);
  n_my = e_hi - e_lo;
  loc_now = el_now > e_lo ? std::min<u64>(el_now - e_lo, n_my) : 0;
  loc_late = n_my - loc_now;
  if (dp) {
    if (cfg.comm_id.size() != 128)
      throw ValidationError("executor: data-parallel run needs the job's 128-byte communicator id (rank 0 draws it)");
    if (W > 8) throw ValidationError("executor: peer-memory data parallelism covers one node (world <= 8)");
    peer = std::make_unique<PeerComm>(R, W, cfg.comm_id, cfg.device);
  }

  cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
  (void)cudaGetLastError();  // do not inherit a stale error of an earlier, unrelated call
  // Stream priorities: the compute stream carries the critical path (the
  // dgrad -> LN' -> attention' chain); the optimizer stream's Adam kernels
  // fill idle SMs (measured +0.5% over default priorities, within run-to-run
  // noise, profiles/round1_stream_prio_ab.txt).
  int prio_lo = 0, prio_hi = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&s_gpu, cudaStreamNonBlocking, prio_hi), "stream");
  cuda_check(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithPriority(&s_opt, cudaStreamNonBlocking, prio_lo), "stream");
  cuda_check(cudaStreamCreateWithFlags(&s_opt_up, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&s_opt_dn, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&ev_opt_begin, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_opt_end, cudaEventDisableTiming), "event");

  // ---- optimizer tier placement
  const u64 opt_bytes = 12 * Ps;  // this rank's shard of the layer's [master, m, v]
  const u64 cpu_opt = cpu_portion(opt_bytes, plan.split.x_opt);
  if (static_cast<int>(cfg.opt_tier) < 0 || static_cast<int>(cfg.opt_tier) > 3)
    throw ValidationError("executor: opt_tier must be 0 (auto), 1 (HBM), 2 (stream) or 3 (host)");
  bool opt_hbm = cfg.opt_tier == OptTier::Hbm;
  host_step = cfg.opt_tier == OptTier::Host;
  size_t free_b = 0, total_b = 0;
  cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  if (cfg.opt_tier == OptTier::Auto) {
    // leave room for params, grads, activations and staging: 3/4 of free HBM
    opt_hbm = static_cast<double>(cpu_opt) * N < 0.6 * static_cast<double>(free_b);
  }

  // ---- device buffers
  const u64 lpb = static_cast<u64>(d.lp());
  for (int i = 0; i < 2; ++i) dev_param[i] = dmalloc(lpb * Ps * static_cast<u64>(W));  // gathered layer
  // Gradient ring (vertical): layer l accumulates into slot l % grad_ring,
  // which the immediate optimizer step of layer l + grad_ring (plan stage
  // +2 after its backward) must have consumed first — a WAR edge of the
  // hazard pass.  Three slots leave that step one stage of slack; when the
  // step streams its state over PCIe it needs more, so the ring takes up to
  // 8 slots within 10% of free HBM.
  if (horizontal) {
    grad_ring = 2;
  } else {
    const double slot = 4.0 * static_cast<double>(Ps) * W;
    grad_ring = static_cast<int>(std::clamp(0.10 * static_cast<double>(free_b) / slot, 3.0, 8.0));
    grad_ring = std::min(grad_ring, std::max(3, N));
  }
  for (int i = 0; i < grad_ring; ++i) {
    grad_slot.push_back(static_cast<float*>(dmalloc(4 * Ps * static_cast<u64>(W))));
    cuda_check(cudaMemset(grad_slot.back(), 0, 4 * Ps * static_cast<u64>(W)), "memset");  // shard padding
    grad_shard.push_back(dp ? static_cast<float*>(dmalloc(4 * Ps)) : grad_slot.back());
  }
  retain.assign(static_cast<size_t>(N), nullptr);
  if (loc_late > 0 && !host_step)
    for (int l = 0; l < N; ++l) retain[static_cast<size_t>(l)] = static_cast<float*>(dmalloc(4 * loc_late));
  n_fixed = static_cast<long long>(d.V + d.s) * d.h;
  fx_master = static_cast<float*>(dmalloc(4 * n_fixed));
  fx_m = static_cast<float*>(dmalloc(4 * n_fixed));
  fx_v = static_cast<float*>(dmalloc(4 * n_fixed));
  fx_grad = static_cast<float*>(dmalloc(4 * n_fixed));
  fx_lp = dmalloc(static_cast<u64>(n_fixed) * d.lp());
  if (dp) {
    fx_shard = (n_fixed + W - 1) / W;
    fx_red = static_cast<float*>(dmalloc(4 * static_cast<u64>(fx_shard)));
    for (int i = 0; i < 2; ++i) pb_param[i] = peer->add(dev_param[i]);
    for (float* g : grad_slot) pb_grad.push_back(peer->add(g));
    pb_fx_grad = peer->add(fx_grad);
    pb_fx_red = peer->add(fx_red);
    peer->connect();
    cuda_check(cudaStreamCreateWithPriority(&s_ag, cudaStreamNonBlocking, prio_hi), "stream");
    cuda_check(cudaStreamCreateWithPriority(&s_rs, cudaStreamNonBlocking, prio_hi), "stream");
    for (cudaEvent_t* e : {&ev_ag[0], &ev_ag[1], &ev_h2d_chunk, &ev_bwd_done})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    ev_rs.assign(static_cast<size_t>(grad_ring), nullptr);
    for (auto& e : ev_rs) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    grad_last.assign(static_cast<size_t>(grad_ring), 0);
  }
  if (!alloc_workspace(d, ws)) throw InfeasibleError("executor: device workspace allocation failed");
  if (cfg.profile_kernels) ws.prof = &prof;
  dev_bytes += ws.bytes;
  for (int i = 0; i < 2 * M; ++i) {
    in_x.push_back(dmalloc(cb));
    out_y.push_back(dmalloc(cb));
    in_g.push_back(dmalloc(cb));
    out_g.push_back(dmalloc(cb));
  }
  const u64 tok_bytes = 4ull * M * d.b * (d.s + 1);
  for (int i = 0; i < 2; ++i) dev_tok[i] = static_cast<int32_t*>(dmalloc(tok_bytes));
  dev_bad_tokens = static_cast<int*>(dmalloc(sizeof(int)));
  cuda_check(cudaMemset(dev_bad_tokens, 0, sizeof(int)), "memset");
  // 2 Mi elements per chunk: 24 MB of state (~0.5 ms of PCIe per direction)
  chunk = static_cast<long long>(std::min<u64>(P, 2ull << 20));
  chunk = (chunk + 3) / 4 * 4;
  for (OptSlot& o : oring) {
    o.state = static_cast<float*>(dmalloc(12ull * chunk));
    o.lp = dmalloc(static_cast<u64>(chunk) * d.lp());
    for (cudaEvent_t* e : {&o.up, &o.comp, &o.free_})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  }
  cuda_check(cudaMemset(fx_m, 0, 4 * n_fixed), "memset");
  cuda_check(cudaMemset(fx_v, 0, 4 * n_fixed), "memset");
  cuda_check(cudaMemset(fx_grad, 0, 4 * n_fixed), "memset");

  // ---- host tiers
  const bool need_nvme = plan.split.x_param < 1.0 || plan.split.x_ckpt < 1.0 || plan.split.x_opt < 1.0;
  if (need_nvme) nvme = std::make_unique<NvmeFile>(cfg.nvme_dir, cfg.odirect, 8);
  const u64 lp = static_cast<u64>(d.lp());
  ring_k = std::max(1, std::min(cfg.ssd_ring_layers, N));
  ring_param.assign(static_cast<size_t>(ring_k), nullptr);
  ring_opt.assign(static_cast<size_t>(ring_k), nullptr);
  ring_ckpt.assign(static_cast<size_t>(ring_k) * M, nullptr);
  // Placement of a layer's params / optimizer state, the reference's byte
  // model (schedule.cpp:309-314): the SSD-resident bytes are ssd_portion of
  // the whole, and the delayed alpha slice owns scaled_portion(ssd, alpha) of
  // them, the immediate slice the rest.  Each slice keeps its CPU part first
  // and its SSD bytes at its end, so every plan SSD transfer of a slice moves
  // exactly that slice's bytes (a single CPU/SSD cut over the whole blob put
  // the delayed slice entirely on the SSD: 2x the plan's bytes in the
  // forward-phase reads and writes, 0.75x in the backward's).
  auto slice_ssd = [&](u64 size, u64 elem_bytes, double x) {
    const u64 e = elem_bytes * loc_now;  // immediate | delayed element boundary
    const u64 ssd = ssd_portion(size, x);
    // one rank: exactly the plan's bytes; ZeRO-3 shards: each rank's delayed
    // elements carry the layer's CPU/SSD proportion (a shard's share of the
    // delayed slice is not alpha)
    u64 late = W == 1 ? scaled_portion(ssd, plan.kind.delay_ratio)
                      : static_cast<u64>(std::llround(static_cast<double>(ssd) * static_cast<double>(size - e) /
                                                      static_cast<double>(std::max<u64>(size, 1))));
    late = std::min(late, size - e);
    u64 now = ssd - late;
    if (now > e) {  // byte rounding at x ~ 0: at most a few bytes move across
      now = e;
      late = ssd - now;
    }
    return std::vector<std::pair<u64, u64>>{{e - now, e}, {size - late, size}};
  };
  for (int l = 0; l < N; ++l) {
    param_blob.push_back(make_blob(lp * Ps, slice_ssd(lp * Ps, lp, plan.split.x_param), false, ring_param, l % ring_k));
    opt_blob.push_back(make_blob(opt_bytes, slice_ssd(opt_bytes, 12, plan.split.x_opt), opt_hbm, ring_opt, l % ring_k));
  }
  // GradAccum D2H landing buffers.  The horizontal schedule reads a layer's
  // partial sum back for the next micro-batch, so it keeps one per layer;
  // in the vertical schedule the optimizer consumes the gradient in HBM and
  // the plan's D2H (schedule.cpp:489-494) only has to land somewhere: a
  // two-slot ring (N x 4P of pinned DRAM would be 258 GB at GPT-65B).
  // With the host-core step the landing slot is read by CpuStep (plan stage
  // +1 after the D2H): six slots keep the in-order D2H queue from waiting on
  // a step still reading the slot it wants to overwrite.
  host_grad_ring = horizontal ? N : std::min(N, host_step ? 6 : 2);
  for (int i = 0; i < host_grad_ring; ++i) host_grad.push_back(arena.alloc(4 * Ps));
  if (host_step) {
    host_retain.assign(static_cast<size_t>(N), nullptr);
    if (loc_late > 0)
      for (int l = 0; l < N; ++l) host_retain[static_cast<size_t>(l)] = reinterpret_cast<float*>(arena.alloc(4 * loc_late));
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    // the node's cores are shared by its W ranks (one process per GPU)
    host_pool = std::make_unique<ThreadPool>(cfg.host_threads > 0 ? cfg.host_threads : std::max(1, (hw - 4) / W), 10);
  }
  for (int l = 0; l < N; ++l)
    for (int m = 0; m < M; ++m)
      ckpt_blob.push_back(
          make_blob(cb, {{cpu_portion(cb, plan.split.x_ckpt), cb}}, false, ring_ckpt, (l % ring_k) * M + m));
  auto has_ssd = [](const Blob& b) {
    for (const Segment& sg : b.segs)
      if (sg.tier == Tier::Ssd) return true;
    return false;
  };
  ssd_param = has_ssd(param_blob[0]);
  ssd_opt = has_ssd(opt_blob[0]);
  ssd_ckpt = has_ssd(ckpt_blob[0]);
  for (int i = 0; i < 2 * M; ++i) host_ilg.push_back(arena.alloc(cb));
  if (nvme) nvme->finalize_size();

  init_weights();
  late_ready.reset(new std::atomic<long long>[static_cast<size_t>(N)]);
  late_applied.reset(new std::atomic<long long>[static_cast<size_t>(N)]);
  for (int l = 0; l < N; ++l) {
    late_ready[static_cast<size_t>(l)].store(-1);
    late_applied[static_cast<size_t>(l)].store(-1);
  }
  build_tasks();
  hazards();
  cuda_check(cudaEventCreate(&ev_base), "event");
}

Executor::Impl::~Impl() {
  cudaDeviceSynchronize();
  for (auto& a : ev_done)
    for (cudaEvent_t e : a)
      if (e) cudaEventDestroy(e);
  for (auto& a : ev_start)
    for (cudaEvent_t e : a)
      if (e) cudaEventDestroy(e);
  if (ev_base) cudaEventDestroy(ev_base);
  for (OptSlot& o : oring)
    for (cudaEvent_t e : {o.up, o.comp, o.free_})
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {ev_opt_begin, ev_opt_end})
    if (e) cudaEventDestroy(e);
  free_workspace(ws);
  peer.reset();
  for (cudaEvent_t e : {ev_ag[0], ev_ag[1], ev_h2d_chunk, ev_bwd_done})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_rs)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {s_ag, s_rs})
    if (s) cudaStreamDestroy(s);
  for (void* p : dev_allocs) cudaFree(p);
  for (cudaStream_t s : {s_gpu, s_h2d, s_d2h, s_opt, s_opt_up, s_opt_dn})
    if (s) cudaStreamDestroy(s);
}

void* Executor::Impl::dmalloc(u64 bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<u64>(bytes, 256)) != cudaSuccess)
    throw InfeasibleError("executor: cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  dev_allocs.push_back(p);
  dev_bytes += bytes;
  return p;
}

// Cut [0,size) at the CPU/SSD boundary and the extra cut points; CPU-resident
// segments live in pinned DRAM (or HBM), SSD segments get an NVMe region and
// a 4 KiB-aligned place in staging slot ring[slot] (allocated by the first
// blob that uses the slot; blobs of one kind have identical segments).
Blob Executor::Impl::make_blob(u64 size, const std::vector<std::pair<u64, u64>>& ssd, bool hbm_for_cpu,
                               std::vector<uint8_t*>& ring, int slot) {
  std::vector<u64> cuts = {0, size};
  for (const auto& r : ssd) {
    cuts.push_back(r.first);
    cuts.push_back(r.second);
  }
  std::sort(cuts.begin(), cuts.end());
  cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
  Blob b;
  b.size = size;
  for (size_t i = 0; i + 1 < cuts.size(); ++i) {
    Segment s;
    s.lo = cuts[i];
    s.hi = cuts[i + 1];
    if (s.hi <= s.lo || s.hi > size) continue;
    bool on_ssd = false;
    for (const auto& r : ssd) on_ssd = on_ssd || (s.lo >= r.first && s.hi <= r.second);
    if (!on_ssd) {
      s.tier = hbm_for_cpu ? Tier::Hbm : Tier::Dram;
      if (hbm_for_cpu) {
        s.dev = static_cast<uint8_t*>(dmalloc(s.size()));
      } else {
        s.img = arena.alloc(s.size());
      }
    } else {
      s.tier = Tier::Ssd;
      s.file_off = nvme->reserve(s.size());
    }
    b.segs.push_back(s);
  }
  u64 staged = 0;
  for (const Segment& s : b.segs)
    if (s.tier == Tier::Ssd) staged += align_up(s.size(), kNvmeAlign);
  if (staged > 0) {
    uint8_t*& base = ring[static_cast<size_t>(slot)];
    if (!base) base = arena.alloc(staged);
    u64 off = 0;
    for (Segment& s : b.segs) {
      if (s.tier != Tier::Ssd) continue;
      s.img = s.rd = base + off;
      off += align_up(s.size(), kNvmeAlign);
    }
  }
  return b;
}

// Initial master weights (fp32) -> optimizer blobs (AoS [master, m=0, v=0]),
// low-precision copies -> parameter blobs; SSD segments persisted to NVMe.
void Executor::Impl::init_weights() {
  const long long h2 = 1LL * d.h * d.h;
  const double scaled = 0.02 / std::sqrt(2.0 * N);
  std::vector<float> state(3 * Ps, 0.0f);  // this rank's shard, padding zero
  std::vector<uint8_t> lpbuf(static_cast<size_t>(d.lp()) * Ps, 0);
  for (int l = 0; l < N; ++l) {
    const uint64_t key = stream_key(cfg.seed, 100 + static_cast<uint64_t>(l));
    parallel_for(static_cast<long long>(n_my), [&](long long lo, long long hi) {
      for (long long i = lo; i < hi; ++i) {
        const long long gi = static_cast<long long>(e_lo) + i;  // element index within the layer
        const bool out_proj = (gi >= 3 * h2 && gi < 4 * h2) || gi >= 8 * h2;
        const float v = static_cast<float>((out_proj ? scaled : 0.02) * normal_at(key, static_cast<uint64_t>(gi)));
        state[3 * static_cast<size_t>(i)] = v;
        state[3 * static_cast<size_t>(i) + 1] = 0.0f;
        state[3 * static_cast<size_t>(i) + 2] = 0.0f;
        if (d.dt == DType::BF16) {
          const uint16_t bv = f32_to_bf16(v);
          std::memcpy(&lpbuf[2 * static_cast<size_t>(i)], &bv, 2);
        } else {
          std::memcpy(&lpbuf[4 * static_cast<size_t>(i)], &v, 4);
        }
      }
    });
    for (Blob* b : {&param_blob[static_cast<size_t>(l)], &opt_blob[static_cast<size_t>(l)]}) {
      const uint8_t* src = b == &param_blob[static_cast<size_t>(l)] ? lpbuf.data()
                                                                    : reinterpret_cast<const uint8_t*>(state.data());
      for (Segment& s : b->segs) {
        if (s.tier == Tier::Hbm) {
          cuda_check(cudaMemcpy(s.dev, src + s.lo, s.size(), cudaMemcpyHostToDevice), "init H2D");
        } else {
          std::memcpy(s.img, src + s.lo, s.size());
          if (s.tier == Tier::Ssd) nvme->write(s.file_off, s.img, s.size());
        }
      }
    }
  }
  // fixed params: wte N(0,0.02) stream 1, wpe stream 2
  std::vector<float> fx(static_cast<size_t>(n_fixed));
  const long long nw = 1LL * d.V * d.h;
  const uint64_t k1 = stream_key(cfg.seed, 1), k2 = stream_key(cfg.seed, 2);
  parallel_for(n_fixed, [&](long long lo, long long hi) {
    for (long long i = lo; i < hi; ++i)
      fx[static_cast<size_t>(i)] = static_cast<float>(
          0.02 * (i < nw ? normal_at(k1, static_cast<uint64_t>(i)) : normal_at(k2, static_cast<uint64_t>(i - nw))));
  });
  cuda_check(cudaMemcpy(fx_master, fx.data(), 4 * n_fixed, cudaMemcpyHostToDevice), "init fixed");
  cuda_check(gs::cast_from_f32(d.dt, fx_master, fx_lp, n_fixed, s_gpu), "cast fixed");
  cuda_check(cudaStreamSynchronize(s_gpu), "init sync");
}

void Executor::Impl::build_tasks() {
  const size_t n = plan.tasks.size();
  res_of.resize(n);
  fwd_phase.assign(n, 0);
  chunk_lo.assign(n, 0);
  {
    // The backward loop (schedule.cpp:431) starts with layer N-1's parameter
    // fetch: its SSD read at stage N-2 or, without SSD bytes, its first PCIe
    // chunk at stage N-1 (the forward fetched layer N-1 at stages N-3 / N-2).
    // Everything emitted earlier is forward-phase, including the delayed
    // slice of the previous iteration's optimizer step.
    bool fwd = true;
    std::map<std::pair<int, int>, u64> next_lo;  // (layer, stage) -> running chunk offset
    for (size_t i = 0; i < n; ++i) {
      const Task& t = plan.tasks[i];
      if (horizontal) fwd = false;  // no delayed slice; every SSD read refreshes the whole tier
      if (fwd && t.kind == TaskKind::Xfer && t.data == DataKind::Param && t.layer == N - 1 &&
          ((t.link == LinkKind::SSD_Read && t.stage == N - 2) || (t.link == LinkKind::PCIe_H2D && t.stage == N - 1)))
        fwd = false;
      fwd_phase[i] = fwd ? 1 : 0;
      if (t.kind == TaskKind::Xfer && t.data == DataKind::Param && t.link == LinkKind::PCIe_H2D) {
        u64& lo = next_lo[{t.layer, t.stage}];
        chunk_lo[i] = lo;
        lo += t.bytes;
      }
    }
  }
  queue.assign(kNumResources, {});
  is_stream.assign(n, 0);
  ev_done.resize(n);
  done_iter = std::vector<std::atomic<int>>(n);
  for (size_t i = 0; i < n; ++i) {
    const Task& t = plan.tasks[i];
    const Resource r = task_resource(t, true);
    res_of[i] = r;
    queue[static_cast<size_t>(r)].push_back(static_cast<int>(i));
    is_stream[i] = (r == Resource::GPU || (r == Resource::CPU && !host_step) || r == Resource::H2D ||
                    r == Resource::D2H) ? 1 : 0;
    done_iter[i].store(-1);
    for (auto& e : ev_done[i]) {
      e = nullptr;
      if (is_stream[i]) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
  }
  if (cfg.record_trace) {
    ev_start.resize(n);
    for (size_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) {
        ev_start[i][static_cast<size_t>(k)] = nullptr;
        if (is_stream[i]) {
          cudaEventDestroy(ev_done[i][static_cast<size_t>(k)]);
          cuda_check(cudaEventCreate(&ev_done[i][static_cast<size_t>(k)]), "event");
          cuda_check(cudaEventCreate(&ev_start[i][static_cast<size_t>(k)]), "event");
        }
      }
  }
}

// ---------------------------------------------------------------- hazards
namespace {
enum SlotKind {
  kDevParam, kInX, kOutY, kInG, kOutG, kGrad, kRetain, kHostIlg, kParamImg, kParamRd, kOptImg, kOptRd, kCkptImg,
  kCkptRd, kHostGrad, kOptDev, kParamFile, kOptFile, kCkptFile, kHostRetain,
  kParamStage, kOptStage, kCkptStage  // SSD staging-ring slots (layer % ring)
};
struct Access {
  long long slot;
  bool write;
};
long long slot_id(int kind, long long a, long long b = 0) { return (static_cast<long long>(kind) << 48) | (a << 24) | b; }
}  // namespace

void Executor::Impl::hazards() {
  const size_t n = plan.tasks.size();
  std::vector<std::vector<Access>> acc(n);
  for (size_t i = 0; i < n; ++i) {
    const Task& t = plan.tasks[i];
    auto R = [&](long long s) { acc[i].push_back({s, false}); };
    auto W = [&](long long s) { acc[i].push_back({s, true}); };
    const int l = t.layer, m = t.microbatch, st = t.stage;
    const int par = ((st % 2) + 2) % 2;
    const int parm1 = (((st - 1) % 2) + 2) % 2;
    const bool late = delayed(t);
    const int imm_late = late ? 1 : 0;
    const int rl = ((l % ring_k) + ring_k) % ring_k, rlm1 = (((l - 1) % ring_k) + ring_k) % ring_k;
    // staging-ring accesses, only for kinds that have SSD-resident bytes
    auto RS = [&](bool on, int kind, long long a, long long b2) {
      if (on) R(slot_id(kind, a, b2));
    };
    auto WS = [&](bool on, int kind, long long a, long long b2) {
      if (on) W(slot_id(kind, a, b2));
    };
    switch (t.kind) {
      case TaskKind::FixedOps: break;
      case TaskKind::FwdCompute:
        R(slot_id(kDevParam, par));
        if (horizontal) {  // activation carried in HBM layer to layer; input staged for the ckpt D2H
          if (l > 0) R(slot_id(kInG, parm1, 0));
          W(slot_id(kInG, par, 0));
          W(slot_id(kOutY, par, 0));
          break;
        }
        if (l > 0) R(m == first_mb(st) ? slot_id(kOutY, parm1, m) : slot_id(kInX, par, m));
        W(slot_id(kOutY, par, m));
        break;
      case TaskKind::RecomputeAndBwd:
        R(slot_id(kDevParam, par));
        if (horizontal) {
          R(slot_id(kInX, par, 0));
          if (l < N - 1) R(slot_id(kOutG, parm1, 0));
          W(slot_id(kOutG, par, 0));
          R(slot_id(kGrad, l % grad_ring));
          W(slot_id(kGrad, l % grad_ring));
          break;
        }
        if (l > 0) R(slot_id(kInX, par, m));
        if (l < N - 1) R(m == first_mb(st) ? slot_id(kOutG, parm1, m) : slot_id(kInG, par, m));
        W(slot_id(kOutG, par, m));
        R(slot_id(kGrad, l % grad_ring));
        W(slot_id(kGrad, l % grad_ring));
        if (m == last_mb(st) && el_late > 0) W(slot_id(kRetain, l));
        break;
      case TaskKind::CpuStep:
        if (host_step) R(late ? slot_id(kHostRetain, l) : slot_id(kHostGrad, l % host_grad_ring));
        else R(late ? slot_id(kRetain, l) : slot_id(kGrad, l % grad_ring));
        R(slot_id(kOptRd, l, imm_late));
        R(slot_id(kOptImg, l, imm_late));
        W(slot_id(kOptImg, l, imm_late));
        W(slot_id(kOptDev, l, imm_late));
        W(slot_id(kParamImg, l));
        RS(ssd_opt, kOptStage, rl, imm_late);
        WS(ssd_opt, kOptStage, rl, imm_late);
        WS(ssd_param, kParamStage, rl, imm_late);
        // a skipped delayed step refills the slice from the file
        if (late) RS(ssd_param, kParamFile, l, 1);
        break;
      case TaskKind::Xfer: {
        const bool fwd = fwd_phase[i] != 0;
        switch (t.data) {
          case DataKind::Param:
            if (t.link == LinkKind::SSD_Read) {
              W(slot_id(kParamRd, l));
              R(slot_id(kParamFile, l, 0));
              WS(ssd_param, kParamStage, rl, 0);
              if (!fwd) {
                R(slot_id(kParamFile, l, 1));
                WS(ssd_param, kParamStage, rl, 1);
              }
            } else if (t.link == LinkKind::SSD_Write) {
              R(slot_id(kParamImg, l));
              W(slot_id(kParamFile, l, imm_late));
              RS(ssd_param, kParamStage, rl, imm_late);
            } else {
              R(slot_id(kParamImg, l));
              R(slot_id(kParamRd, l));
              RS(ssd_param, kParamStage, rl, 0);
              RS(ssd_param, kParamStage, rl, 1);
              W(slot_id(kDevParam, (((st + 1) % 2) + 2) % 2));
            }
            break;
          case DataKind::Ckpt:
            if (horizontal) {  // checkpoint (l, m) = the INPUT of layer l (schedule.cpp:186-209)
              if (t.link == LinkKind::PCIe_D2H) {
                R(slot_id(kOutY, par, 0));
                W(slot_id(kCkptImg, l, m));
                WS(ssd_ckpt, kCkptStage, rl, m);
              } else if (t.link == LinkKind::PCIe_H2D) {
                R(slot_id(kCkptImg, l, m));
                R(slot_id(kCkptRd, l, m));
                RS(ssd_ckpt, kCkptStage, rl, m);
                W(slot_id(kInX, par, 0));
              } else if (t.link == LinkKind::SSD_Write) {
                R(slot_id(kCkptImg, l, m));
                W(slot_id(kCkptFile, l, m));
                RS(ssd_ckpt, kCkptStage, rl, m);
              } else {
                W(slot_id(kCkptRd, l, m));
                R(slot_id(kCkptFile, l, m));
                WS(ssd_ckpt, kCkptStage, rl, m);
              }
              break;
            }
            if (t.link == LinkKind::PCIe_D2H) {
              R(slot_id(kOutY, par, m));
              W(slot_id(kCkptImg, l, m));
              WS(ssd_ckpt, kCkptStage, rl, m);
            } else if (t.link == LinkKind::PCIe_H2D) {
              R(slot_id(kCkptImg, l - 1, m));
              if (!fwd) R(slot_id(kCkptRd, l - 1, m));
              RS(ssd_ckpt, kCkptStage, rlm1, m);
              W(slot_id(kInX, par, m));
            } else if (t.link == LinkKind::SSD_Write) {
              for (int k = 0; k < M; ++k) {
                R(slot_id(kCkptImg, l, k));
                W(slot_id(kCkptFile, l, k));
                RS(ssd_ckpt, kCkptStage, rl, k);
              }
            } else {
              for (int k = 0; k < M; ++k) {
                W(slot_id(kCkptRd, l - 1, k));
                R(slot_id(kCkptFile, l - 1, k));
                WS(ssd_ckpt, kCkptStage, rlm1, k);
              }
            }
            break;
          case DataKind::GradAccum:
            if (t.link == LinkKind::PCIe_D2H) {
              R(slot_id(kGrad, l % grad_ring));
              W(slot_id(kHostGrad, l % host_grad_ring));
              if (host_step && loc_late > 0) W(slot_id(kHostRetain, l));
            } else {  // horizontal accumulation fetch
              R(slot_id(kHostGrad, l % host_grad_ring));
              W(slot_id(kGrad, l % grad_ring));
            }
            break;
          case DataKind::InterlayerGrad:
            if (t.link == LinkKind::PCIe_D2H) {
              R(slot_id(kOutG, par, m));
              W(slot_id(kHostIlg, par, m));
            } else {
              R(slot_id(kHostIlg, parm1, m));
              W(slot_id(kInG, par, m));
            }
            break;
          case DataKind::OptState:
            if (t.link == LinkKind::SSD_Read) {
              W(slot_id(kOptRd, l, imm_late));
              R(slot_id(kOptFile, l, imm_late));
              WS(ssd_opt, kOptStage, rl, imm_late);
            } else {
              R(slot_id(kOptImg, l, imm_late));
              W(slot_id(kOptFile, l, imm_late));
              RS(ssd_opt, kOptStage, rl, imm_late);
            }
            break;
        }
        break;
      }
    }
  }
  // RAW / WAR / WAW over two unrolled iterations; deps discovered in
  // iteration 1 carry offsets 0 / -1 and hold in every steady-state
  // iteration.  RAW edges matter where data flows through a buffer the plan
  // does not name: e.g. the next iteration's parameter SSD read must follow
  // this iteration's SSD write-back of the updated slice (same NVMe region).
  struct Use {
    int task, iter;
  };
  std::map<long long, std::vector<Use>> readers;
  std::map<long long, Use> writer;
  std::vector<std::set<std::pair<int, int>>> found(n);
  for (int it = 0; it < 2; ++it) {
    for (size_t i = 0; i < n; ++i) {
      for (const Access& a : acc[i]) {
        if (a.write) continue;
        readers[a.slot].push_back({static_cast<int>(i), it});
        auto w = writer.find(a.slot);
        if (w != writer.end() && !(w->second.task == static_cast<int>(i) && w->second.iter == it) && it == 1)
          found[i].insert({w->second.task, w->second.iter - it});
      }
      for (const Access& a : acc[i]) {
        if (!a.write) continue;
        auto add = [&](Use u) {
          if (u.task == static_cast<int>(i) && u.iter == it) return;
          if (it == 1) found[i].insert({u.task, u.iter - it});
        };
        for (const Use& u : readers[a.slot]) add(u);
        auto w = writer.find(a.slot);
        if (w != writer.end()) add(w->second);
        readers[a.slot].clear();
        writer[a.slot] = {static_cast<int>(i), it};
      }
    }
  }
  extra.assign(n, {});
  for (size_t i = 0; i < n; ++i) {
    const Task& t = plan.tasks[i];
    for (const auto& [task, offv] : found[i]) {
      if (offv == 0 && std::binary_search(t.deps.begin(), t.deps.end(), task)) continue;
      if (offv == -1 && t.cross_iter_dep == task) continue;
      if (res_of[static_cast<size_t>(task)] == res_of[i] && offv == 0 && task < static_cast<int>(i)) continue;  // FIFO order
      extra[i].push_back({task, offv});
    }
  }
}

// ------------------------------------------------------------ data movement
// Upload logical bytes [lo,hi) of a blob to dst.  SSD segments come from the
// read staging (Src::ReadStaging), the image (Src::Image) or, for Auto, the
// image when the segment lies at/after `delayed_lo` (freshly produced by the
// delayed step) and the staging otherwise.  Returns bytes moved over PCIe.
u64 Executor::Impl::upload(const Blob& b, u64 lo, u64 hi, void* dst, Src src, cudaStream_t st, u64 delayed_lo) {
  u64 moved = 0;
  for (const Segment& s : b.segs) {
    const u64 a = std::max(lo, s.lo), e = std::min(hi, s.hi);
    if (a >= e) continue;
    const uint8_t* from;
    cudaMemcpyKind kind = cudaMemcpyHostToDevice;
    if (s.tier == Tier::Hbm) {
      from = s.dev;
      kind = cudaMemcpyDeviceToDevice;
    } else if (s.tier == Tier::Dram) {
      from = s.img;
    } else {
      const bool img = src == Src::Image || (src == Src::Auto && s.lo >= delayed_lo);
      from = img ? s.img : s.rd;
    }
    cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + (a - lo), from + (a - s.lo), e - a, kind, st), "upload");
    if (kind == cudaMemcpyHostToDevice) moved += e - a;
  }
  return moved;
}

u64 Executor::Impl::download(Blob& b, u64 lo, u64 hi, const void* src, cudaStream_t st) {
  u64 moved = 0;
  for (Segment& s : b.segs) {
    const u64 a = std::max(lo, s.lo), e = std::min(hi, s.hi);
    if (a >= e) continue;
    const uint8_t* from = static_cast<const uint8_t*>(src) + (a - lo);
    if (s.tier == Tier::Hbm) {
      if (s.dev + (a - s.lo) != from)
        cuda_check(cudaMemcpyAsync(s.dev + (a - s.lo), from, e - a, cudaMemcpyDeviceToDevice, st), "download");
    } else {
      cuda_check(cudaMemcpyAsync(s.img + (a - s.lo), from, e - a, cudaMemcpyDeviceToHost, st), "download");
      moved += e - a;
    }
  }
  return moved;
}

// NVMe write (image -> file) or read (file -> staging) of the SSD segments
// overlapping [lo,hi).  Whole segments move (they are the I/O units).
u64 Executor::Impl::ssd_io(Blob& b, u64 lo, u64 hi, bool write) {
  u64 phys = 0;
  for (Segment& s : b.segs) {
    if (s.tier != Tier::Ssd || s.hi <= lo || s.lo >= hi) continue;
    phys += write ? nvme->write(s.file_off, s.img, s.size()) : nvme->read(s.file_off, s.rd, s.size());
  }
  return phys;
}

// ------------------------------------------------------------ execution
cudaStream_t Executor::Impl::stream_of(Resource r) const {
  switch (r) {
    case Resource::GPU: return s_gpu;
    case Resource::CPU: return s_opt;
    case Resource::H2D: return s_h2d;
    case Resource::D2H: return s_d2h;
    default: return nullptr;
  }
}

void Executor::Impl::wait_dep(int dep, int iter, bool on_stream, cudaStream_t st) {
  if (iter < 0) return;
  {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return done_iter[static_cast<size_t>(dep)].load() >= iter || failed.load(); });
  }
  if (failed.load()) throw std::runtime_error("aborted");
  if (!is_stream[static_cast<size_t>(dep)]) return;
  cudaEvent_t e = ev_done[static_cast<size_t>(dep)][static_cast<size_t>(iter % 3)];
  if (on_stream)
    cuda_check(cudaStreamWaitEvent(st, e, 0), "cudaStreamWaitEvent");
  else
    cuda_check(cudaEventSynchronize(e), "cudaEventSynchronize");
}

void Executor::Impl::note_ledger(int it, const Task& t, u64 phys) {
  std::lock_guard<std::mutex> g(led_mu);
  if (it != last_iter) return;
  led_logical.at(t.link, t.data) += t.bytes;
  led_phys.at(t.link, t.data) += phys;
}
void Executor::Impl::note_ext(int it, LinkKind l, DataKind dk, u64 bytes) {
  if (bytes == 0) return;
  std::lock_guard<std::mutex> g(led_mu);
  if (it != last_iter) return;
  led_ext.at(l, dk) += bytes;
}

void Executor::Impl::run_task(int id, int it) {
  const Task& t = plan.tasks[static_cast<size_t>(id)];
  const Resource r = res_of[static_cast<size_t>(id)];
  const bool stream = is_stream[static_cast<size_t>(id)];
  cudaStream_t st = stream_of(r);
  const auto w0 = std::chrono::steady_clock::now();
  for (int dep : t.deps) wait_dep(dep, it, stream, st);
  if (t.cross_iter_dep >= 0) wait_dep(t.cross_iter_dep, it - 1, stream, st);
  for (const ExtraDep& x : extra[static_cast<size_t>(id)]) wait_dep(x.task, it + x.offset, stream, st);

  const auto h0 = std::chrono::steady_clock::now();
  if (stream && cfg.record_trace)
    cuda_check(cudaEventRecord(ev_start[static_cast<size_t>(id)][static_cast<size_t>(it % 3)], st), "record");
  u64 phys = 0;
  switch (t.kind) {
    case TaskKind::FwdCompute:
    case TaskKind::RecomputeAndBwd:
    case TaskKind::FixedOps: compute_task(t, it); break;
    case TaskKind::CpuStep: step_task(t, it); break;
    case TaskKind::Xfer: xfer_task(t, it, phys); break;
  }
  if (stream) {
    cuda_check(cudaEventRecord(ev_done[static_cast<size_t>(id)][static_cast<size_t>(it % 3)], st), "record");
  }
  if (host_prof && r == Resource::GPU) {
    const auto h1 = std::chrono::steady_clock::now();
    host_wait_s += std::chrono::duration<double>(h0 - w0).count();
    host_enqueue_s += std::chrono::duration<double>(h1 - h0).count();
  }
  if (t.kind == TaskKind::Xfer) note_ledger(it, t, phys);
  if (cfg.record_trace) {
    TraceRecord rec{it, id, r, 0.0, 0.0, t.bytes, phys,
                    std::chrono::duration<double, std::milli>(h0 - host_base).count()};
    if (!stream) {
      rec.t_start_ms = std::chrono::duration<double, std::milli>(h0 - host_base).count();
      rec.t_end_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_base).count();
    }
    std::lock_guard<std::mutex> g(trace_mu);
    trace.push_back(rec);
  }
  {
    std::lock_guard<std::mutex> g(mu);
    done_iter[static_cast<size_t>(id)].store(it);
  }
  cv.notify_all();
}

void Executor::Impl::compute_task(const Task& t, int it) {
  const long long git = global_iter + it;
  const int slot = static_cast<int>(git % 2);
  LaunchCounter lc;
  if (t.kind == TaskKind::FixedOps) {
    const long long tok_n = 1LL * M * d.b * (d.s + 1);
    // token ids of this iteration: host tokens are read from the mapped
    // pinned buffer by an SM copy kernel (a cudaMemcpy would queue on the
    // copy engines behind the plan's bulk parameter / checkpoint DMA)
    const int32_t* src = run_tokens + static_cast<long long>(it) * tok_n;
    const int32_t* from = src;
    if (!run_tokens_dev) {
      void* dp = nullptr;
      cuda_check(cudaHostGetDevicePointer(&dp, const_cast<int32_t*>(src), 0), "token device pointer");
      from = static_cast<const int32_t*>(dp);
    }
    cuda_check(gs::copy_tokens(dev_tok[slot], from, tok_n, d.V, dev_bad_tokens, s_gpu), "tokens");
    lc.n += 1;
    cuda_check(cudaMemsetAsync(dev_loss + it, 0, sizeof(double), s_gpu), "loss");
    if (fixed_done < git) {  // embedding / head step with the previous iteration's grads
      if (dp) {
        fixed_allreduce(s_gpu);
        lc.n += 5;  // four counter signals + the sum
      }
      gs::AdamHyper hp{cfg.adam.lr, cfg.adam.beta1, cfg.adam.beta2, cfg.adam.eps, cfg.adam.weight_decay};
      cuda_check(gs::adam_step(hp, static_cast<int>(git), 1.0f, fx_master, fx_m, fx_v, fx_grad, fx_lp, d.dt, n_fixed,
                               s_gpu),
                 "fixed adam");
      cuda_check(cudaMemsetAsync(fx_grad, 0, 4 * n_fixed, s_gpu), "fixed grad");
      fixed_done = git;
      lc.n += 1;
    }
    launches += lc.n;
    return;
  }
  const int l = t.layer, m = t.microbatch, st = t.stage;
  const int par = st % 2, parm1 = (st + 1) % 2;
  const long long tok_n = 1LL * d.b * (d.s + 1);
  const int32_t* tok = dev_tok[slot] + m * tok_n;
  const void* Wt = dev_param[par];
  if (dp && m == first_mb(st)) {
    // first compute of the stage: the peers' shards of the layer were copied
    // chunk by chunk on s_ag as they landed (xfer_task, Param H2D)
    cuda_check(cudaStreamWaitEvent(s_gpu, ev_ag[par], 0), "gather wait");
  }
  const void* wte = fx_lp;
  const void* wpe = static_cast<const uint8_t*>(fx_lp) + 1LL * d.V * d.h * d.lp();
  auto ck = [&](std::vector<void*>& v, int p, int mb) { return v[static_cast<size_t>(p * M + mb)]; };

  if (t.kind == TaskKind::FwdCompute) {
    const void* x;
    if (l == 0) {
      cuda_check(gs::embed_fwd(d.dt, wte, wpe, tok, ws.x0, d.b, d.s, d.h, s_gpu), "embed");
      lc.n += 1;
      x = ws.x0;
    } else if (horizontal) {
      x = ck(in_g, parm1, 0);  // previous layer's output of the same micro-batch
    } else {
      x = m == first_mb(st) ? ck(out_y, parm1, m) : ck(in_x, par, m);
    }
    if (horizontal) {
      // horizontal checkpoints are layer INPUTS (schedule.cpp:186-188): stage a
      // copy for the D2H so the carry buffer can move on
      cuda_check(cudaMemcpyAsync(ck(out_y, par, 0), x, cb, cudaMemcpyDeviceToDevice, s_gpu), "ckpt stage");
      cuda_check(layer_forward(d, Wt, x, ck(in_g, par, 0), ws, s_gpu, lc), "layer_forward");
    } else {
      cuda_check(layer_forward(d, Wt, x, ck(out_y, par, m), ws, s_gpu, lc), "layer_forward");
    }
    launches += lc.n;
    return;
  }

  // RecomputeAndBwd
  float* gslot = grad_slot[static_cast<size_t>(l % grad_ring)];
  const void* x;
  if (l == 0) {
    cuda_check(gs::embed_fwd(d.dt, wte, wpe, tok, ws.x0, d.b, d.s, d.h, s_gpu), "embed");
    lc.n += 1;
    x = ws.x0;
  } else {
    x = horizontal ? ck(in_x, par, 0) : ck(in_x, par, m);
  }
  HeadArgs head;
  const HeadArgs* hp = nullptr;
  const void* dy = nullptr;
  if (l == N - 1) {
    head.wte = wte;
    head.dwte = fx_grad;
    head.tokens = tok;
    head.scale = 1.0f / (static_cast<float>(d.T()) * static_cast<float>(M) * static_cast<float>(W));
    head.loss_sum = dev_loss + it;
    hp = &head;
  } else if (horizontal) {
    dy = ck(out_g, parm1, 0);  // dx of layer l+1, same micro-batch
  } else {
    dy = m == first_mb(st) ? ck(out_g, parm1, m) : ck(in_g, par, m);
  }
  void* dx = horizontal ? ck(out_g, par, 0) : ck(out_g, par, m);
  bool first;
  if (horizontal) first = (m == 0);  // later MBs accumulate onto the fetched partial sum
  else first = (m == first_mb(st));
  if (dp && first) {
    // the slot's previous layer partial must have been read by every peer
    peer->wait(s_gpu, PeerComm::kGradRead, grad_last[static_cast<size_t>(l % grad_ring)]);
  }
  cuda_check(layer_backward(d, Wt, x, dy, dx, gslot, first, hp, ws, s_gpu, lc), "layer_backward");
  if (dp && !horizontal && m == last_mb(st)) {
    // full-layer fp32 gradient of this rank's micro-batches -> summed shard,
    // on s_rs: the next stage's compute does not wait for it
    const size_t k = static_cast<size_t>(l % grad_ring);
    cuda_check(cudaEventRecord(ev_bwd_done, s_gpu), "record");
    cuda_check(cudaStreamWaitEvent(s_rs, ev_bwd_done, 0), "wait");
    const uint32_t g = ++grad_q;
    peer->signal(s_rs, PeerComm::kGradReady, g);
    peer->wait(s_rs, PeerComm::kGradReady, g);
    gs::PeerSrcs src{};
    for (int r = 0; r < W; ++r)
      src.p[r] = static_cast<const float*>(peer->ptr(pb_grad[k], r)) + static_cast<u64>(R) * Ps;
    cuda_check(gs::peer_sum(src, W, grad_shard[k], static_cast<long long>(Ps), s_rs), "reduce-scatter");
    lc.n += 3;  // two counter signals + the sum
    peer->signal(s_rs, PeerComm::kGradRead, g);
    grad_last[k] = g;
  }
  if (l == 0) {
    cuda_check(gs::embed_bwd(d.dt, tok, dx, fx_grad, fx_grad + 1LL * d.V * d.h, d.b, d.s, d.h, s_gpu), "embed_bwd");
    lc.n += 1;
  }
  if (!horizontal && m == last_mb(st) && el_late > 0) {
    if (loc_late > 0 && !host_step)
      cuda_check(cudaMemcpyAsync(retain[static_cast<size_t>(l)], grad_shard[static_cast<size_t>(l % grad_ring)] + loc_now,
                                 4 * loc_late, cudaMemcpyDeviceToDevice, dp ? s_rs : s_gpu),
                 "retain");
    late_ready[static_cast<size_t>(l)].store(git);
  }
  if (dp && !horizontal && m == last_mb(st))
    cuda_check(cudaEventRecord(ev_rs[static_cast<size_t>(l % grad_ring)], s_rs), "record");
  launches += lc.n;
}

// Fused Adam over elements [e0,e1) of layer l on stream st.  State held in
// HBM is updated in place; otherwise each chunk is staged through the slot
// ring: upload (s_opt_up) -> adam_step_packed (st) -> download of the state
// and of the low-precision params to their host images (s_opt_dn), slot
// reuse ordered by the slot's `free_` event.  st joins the last download
// before returning, so an event recorded on st after this call covers all
// of the step's traffic.
void Executor::Impl::apply_adam(int layer, u64 e0, u64 e1, const float* grad, int step, cudaStream_t st, int it,
                                Src src) {
  gs::AdamHyper hp{cfg.adam.lr, cfg.adam.beta1, cfg.adam.beta2, cfg.adam.eps, cfg.adam.weight_decay};
  Blob& ob = opt_blob[static_cast<size_t>(layer)];
  Blob& pbb = param_blob[static_cast<size_t>(layer)];
  const u64 lp = static_cast<u64>(d.lp());
  // the uploads must follow everything already ordered on st (the task's
  // dependencies were enqueued there as stream waits)
  cuda_check(cudaEventRecord(ev_opt_begin, st), "record");
  cuda_check(cudaStreamWaitEvent(s_opt_up, ev_opt_begin, 0), "wait");
  for (u64 c0 = e0; c0 < e1; c0 += static_cast<u64>(chunk)) {
    const u64 c1 = std::min(e1, c0 + static_cast<u64>(chunk));
    const u64 lo = 12 * c0, hi = 12 * c1;
    OptSlot& slot = oring[static_cast<size_t>(oring_next)];
    oring_next = (oring_next + 1) % kOptRing;
    float* state = nullptr;
    for (Segment& s : ob.segs)
      if (s.tier == Tier::Hbm && s.lo <= lo && hi <= s.hi) state = reinterpret_cast<float*>(s.dev + (lo - s.lo));
    const bool in_place = state != nullptr && (reinterpret_cast<uintptr_t>(state) & 15) == 0;
    u64 up = 0, down = 0;
    if (!in_place) {
      if (slot.used) cuda_check(cudaStreamWaitEvent(s_opt_up, slot.free_, 0), "wait");
      state = slot.state;
      up = upload(ob, lo, hi, state, src, s_opt_up, ~0ull);
      cuda_check(cudaEventRecord(slot.up, s_opt_up), "record");
      cuda_check(cudaStreamWaitEvent(st, slot.up, 0), "wait");
    } else if (slot.used) {
      cuda_check(cudaStreamWaitEvent(st, slot.free_, 0), "wait");  // slot.lp reuse
    }
    cuda_check(gs::adam_step_packed(hp, step, 1.0f, state, grad + (c0 - e0), slot.lp, d.dt,
                                    static_cast<long long>(c1 - c0), st),
               "adam");
    launches += 1;
    cuda_check(cudaEventRecord(slot.comp, st), "record");
    cuda_check(cudaStreamWaitEvent(s_opt_dn, slot.comp, 0), "wait");
    if (!in_place) down = download(ob, lo, hi, state, s_opt_dn);
    const u64 pdown = download(pbb, lp * c0, lp * c1, slot.lp, s_opt_dn);
    cuda_check(cudaEventRecord(slot.free_, s_opt_dn), "record");
    slot.used = true;
    note_ext(it, LinkKind::PCIe_H2D, DataKind::OptState, up);
    note_ext(it, LinkKind::PCIe_D2H, DataKind::OptState, down);
    note_ext(it, LinkKind::PCIe_D2H, DataKind::Param, pdown);
  }
  cuda_check(cudaEventRecord(ev_opt_end, s_opt_dn), "record");
  cuda_check(cudaStreamWaitEvent(st, ev_opt_end, 0), "wait");
}

void Executor::Impl::apply_adam_host(int layer, u64 e0, u64 e1, const float* grad, int step) {
  const HostAdamHyper hp{cfg.adam.lr, cfg.adam.beta1, cfg.adam.beta2, cfg.adam.eps, cfg.adam.weight_decay};
  Blob& ob = opt_blob[static_cast<size_t>(layer)];
  Blob& pbb = param_blob[static_cast<size_t>(layer)];
  const u64 lp = static_cast<u64>(d.lp());
  // walk the element range by (opt segment x param segment) pieces: both
  // blobs are cut at the same element boundaries (split rounding aside), so
  // a piece is contiguous in the state image and in the param image
  u64 e = e0;
  while (e < e1) {
    const Segment* so = nullptr;
    for (const Segment& sg : ob.segs)
      if (sg.lo <= 12 * e && 12 * e < sg.hi) so = &sg;
    const Segment* sp = nullptr;
    for (const Segment& sg : pbb.segs)
      if (sg.lo <= lp * e && lp * e < sg.hi) sp = &sg;
    if (!so || !sp) throw PlanBugError("executor: optimizer element outside its blobs");
    if (so->tier == Tier::Hbm) throw PlanBugError("executor: host step over HBM-resident optimizer state");
    // piece end: the nearer segment end (whole elements)
    u64 end = std::min<u64>(e1, std::min<u64>(so->hi / 12, sp->hi / lp));
    if (end <= e) {
      // a segment boundary inside an element (byte-granular split rounding):
      // step that element through a local copy
      float st3[3];
      uint8_t lpb[4];
      for (int k = 0; k < 3; ++k) {
        for (u64 b = 0; b < 4; ++b) {
          const u64 off = 12 * e + 4 * static_cast<u64>(k) + b;
          for (const Segment& sg : ob.segs)
            if (sg.lo <= off && off < sg.hi) reinterpret_cast<uint8_t*>(st3)[4 * k + static_cast<int>(b)] = sg.img[off - sg.lo];
        }
      }
      host_adam_step(hp, step, st3, grad + (e - e0), lpb, static_cast<int>(lp), 1, *host_pool);
      for (u64 b = 0; b < 12; ++b)
        for (Segment& sg : ob.segs)
          if (sg.lo <= 12 * e + b && 12 * e + b < sg.hi) sg.img[12 * e + b - sg.lo] = reinterpret_cast<uint8_t*>(st3)[b];
      for (u64 b = 0; b < lp; ++b)
        for (Segment& sg : pbb.segs)
          if (sg.lo <= lp * e + b && lp * e + b < sg.hi) sg.img[lp * e + b - sg.lo] = lpb[b];
      ++e;
      continue;
    }
    // a piece may start mid-element only where a boundary split an element,
    // which the branch above consumed; both offsets are element-aligned here
    float* state = reinterpret_cast<float*>(so->img + (12 * e - so->lo));
    void* out = sp->img + (lp * e - sp->lo);
    host_adam_step(hp, step, state, grad + (e - e0), out, static_cast<int>(lp), end - e, *host_pool);
    e = end;
  }
}

// Embedding / position gradient all-reduce (FixedOps, flush): reduce-scatter
// over peer memory into this rank's fx_red shard, then all-gather of the
// peers' shards back into fx_grad.  The counters order every cross-rank
// read before the write that would clobber it: fx_red is rewritten only
// after every peer gathered it (kFixedGathered of the previous round), and
// fx_grad only after every peer summed out of it (kFixedReduced).
void Executor::Impl::fixed_allreduce(cudaStream_t st) {
  const uint32_t f = ++fixed_q;
  const long long lo = std::min<long long>(n_fixed, static_cast<long long>(R) * fx_shard);
  const long long n = std::min<long long>(fx_shard, n_fixed - lo);
  peer->wait(st, PeerComm::kFixedGathered, f - 1);
  peer->signal(st, PeerComm::kFixedReady, f);
  peer->wait(st, PeerComm::kFixedReady, f);
  gs::PeerSrcs src{};
  for (int r = 0; r < W; ++r) src.p[r] = static_cast<const float*>(peer->ptr(pb_fx_grad, r)) + lo;
  cuda_check(gs::peer_sum(src, W, fx_red, n, st), "embedding reduce-scatter");
  peer->signal(st, PeerComm::kFixedReduced, f);
  peer->wait(st, PeerComm::kFixedReduced, f);
  for (int r = 0; r < W; ++r) {
    if (r == R) {
      cuda_check(cudaMemcpyAsync(fx_grad + lo, fx_red, 4 * static_cast<u64>(n), cudaMemcpyDeviceToDevice, st), "gather");
      continue;
    }
    const long long rlo = std::min<long long>(n_fixed, static_cast<long long>(r) * fx_shard);
    const long long rn = std::min<long long>(fx_shard, n_fixed - rlo);
    if (rn > 0)
      cuda_check(cudaMemcpyAsync(fx_grad + rlo, peer->ptr(pb_fx_red, r), 4 * static_cast<u64>(rn),
                                 cudaMemcpyDeviceToDevice, st),
                 "embedding gather");
  }
  peer->signal(st, PeerComm::kFixedGathered, f);
}

void Executor::Impl::step_task(const Task& t, int it) {
  const long long git = global_iter + it;
  const int l = t.layer;
  if (delayed(t)) {
    // alpha slice of the previous iteration (step count git); nothing is
    // retained before the first iteration
    const long long ready = late_ready[static_cast<size_t>(l)].load();
    if (el_late == 0 || ready != git - 1 || late_applied[static_cast<size_t>(l)].load() >= ready) {
      // nothing to apply (first iteration, or flushed): the slice's SSD bytes
      // still have to be in the staging slot for the plan's parameter write-
      // back and upload that follow
      if (loc_late > 0 && ssd_param) {
        // the dependencies were enqueued on s_opt as stream waits; this host
        // write into the (shared) staging slot must follow them too
        cuda_check(cudaStreamSynchronize(s_opt), "refill sync");
        const u64 lp = static_cast<u64>(d.lp());
        ssd_io(param_blob[static_cast<size_t>(l)], lp * loc_now, lp * n_my, false);
      }
      return;
    }
    if (loc_late > 0) {
      if (host_step) apply_adam_host(l, loc_now, n_my, host_retain[static_cast<size_t>(l)], static_cast<int>(git));
      else apply_adam(l, loc_now, n_my, retain[static_cast<size_t>(l)], static_cast<int>(git), s_opt, it);
    }
    late_applied[static_cast<size_t>(l)].store(ready);
    return;
  }
  if (loc_now > 0 && host_step)
    apply_adam_host(l, 0, loc_now, reinterpret_cast<const float*>(host_grad[static_cast<size_t>(l % host_grad_ring)]),
                    static_cast<int>(git + 1));
  else if (loc_now > 0)
    apply_adam(l, 0, loc_now, grad_shard[static_cast<size_t>(l % grad_ring)], static_cast<int>(git + 1), s_opt, it);
}

void Executor::Impl::xfer_task(const Task& t, int it, u64& phys) {
  const int l = t.layer, m = t.microbatch, st = t.stage;
  const int par = ((st % 2) + 2) % 2, parm1 = (((st - 1) % 2) + 2) % 2;
  const bool fwd = fwd_phase[static_cast<size_t>(t.id)] != 0;
  const u64 lp = static_cast<u64>(d.lp());
  auto ck = [&](std::vector<void*>& v, int p, int mb) { return v[static_cast<size_t>(p * M + mb)]; };
  switch (t.data) {
    case DataKind::Param: {
      Blob& b = param_blob[static_cast<size_t>(l)];
      if (t.link == LinkKind::SSD_Read) {
        // forward: only the immediate slice is re-read (the delayed slice was
        // just produced in DRAM by the delayed step); backward: all of it
        phys = fwd ? ssd_io(b, 0, lp * loc_now, false) : ssd_io(b, 0, b.size, false);
      } else if (t.link == LinkKind::SSD_Write) {
        phys = delayed(t) ? ssd_io(b, lp * loc_now, b.size, true) : ssd_io(b, 0, lp * loc_now, true);
      } else {
        // chunk j of the layer's params (dp = 1: the shard is the layer),
        // cut by chunk_size(shard, M, j) in emission order
        const u64 lo = chunk_lo[static_cast<size_t>(t.id)];
        const int use_par = (((st + 1) % 2) + 2) % 2;
        const Src src = fwd ? Src::Auto : Src::ReadStaging;
        // the peers must have copied this buffer's previous contents (two
        // stages ago) out of this rank's region before it is overwritten
        if (dp && lo == 0) peer->wait(s_h2d, PeerComm::kParamRead, param_last[use_par]);
        // this rank's shard lands at its offset of the gathered layer buffer
        phys = upload(b, lo, lo + t.bytes, static_cast<uint8_t*>(dev_param[use_par]) + lp * Ps * R + lo, src, s_h2d,
                      lp * loc_now);
        if (dp) {
          // announce the chunk; copy the peers' same chunk once it has landed
          // there (s_ag follows s_h2d, so it inherits the buffer's local
          // WAR ordering against the compute that last read it)
          const uint32_t q = ++param_q;
          peer->signal(s_h2d, PeerComm::kParamReady, q);
          cuda_check(cudaEventRecord(ev_h2d_chunk, s_h2d), "record");
          cuda_check(cudaStreamWaitEvent(s_ag, ev_h2d_chunk, 0), "wait");
          peer->wait(s_ag, PeerComm::kParamReady, q);
          for (int r = 0; r < W; ++r) {
            if (r == R) continue;
            const u64 off = lp * Ps * static_cast<u64>(r) + lo;
            cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(dev_param[use_par]) + off,
                                       static_cast<const uint8_t*>(peer->ptr(pb_param[use_par], r)) + off, t.bytes,
                                       cudaMemcpyDeviceToDevice, s_ag),
                       "gather");
          }
          peer->signal(s_ag, PeerComm::kParamRead, q);
          launches += 2;  // the two counter signals
          cuda_check(cudaEventRecord(ev_ag[use_par], s_ag), "record");
          param_last[use_par] = q;
        }
      }
      break;
    }
    case DataKind::Ckpt: {
      if (horizontal) {
        Blob& b = ckpt_blob[static_cast<size_t>(l * M + m)];
        if (t.link == LinkKind::PCIe_D2H) phys = download(b, 0, cb, ck(out_y, par, 0), s_d2h);
        else if (t.link == LinkKind::PCIe_H2D) phys = upload(b, 0, cb, ck(in_x, par, 0), Src::ReadStaging, s_h2d, ~0ull);
        else if (t.link == LinkKind::SSD_Write) phys = ssd_io(b, 0, cb, true);
        else phys = ssd_io(b, 0, cb, false);
        break;
      }
      if (t.link == LinkKind::PCIe_D2H) {
        phys = download(ckpt_blob[static_cast<size_t>(l * M + m)], 0, cb, ck(out_y, par, m), s_d2h);
      } else if (t.link == LinkKind::PCIe_H2D) {
        phys = upload(ckpt_blob[static_cast<size_t>((l - 1) * M + m)], 0, cb, ck(in_x, par, m),
                      fwd ? Src::Image : Src::ReadStaging, s_h2d, ~0ull);
      } else if (t.link == LinkKind::SSD_Write) {
        for (int k = 0; k < M; ++k) phys += ssd_io(ckpt_blob[static_cast<size_t>(l * M + k)], 0, cb, true);
      } else {
        for (int k = 0; k < M; ++k) phys += ssd_io(ckpt_blob[static_cast<size_t>((l - 1) * M + k)], 0, cb, false);
      }
      break;
    }
    case DataKind::GradAccum: {
      float* g = grad_shard[static_cast<size_t>(l % grad_ring)];
      if (dp && t.link == LinkKind::PCIe_D2H)
        cuda_check(cudaStreamWaitEvent(s_d2h, ev_rs[static_cast<size_t>(l % grad_ring)], 0), "reduce wait");
      if (t.link == LinkKind::PCIe_D2H && host_step) {
        // immediate slice -> the ring slot the step reads, delayed slice ->
        // the layer's retained copy (the next iteration's forward-phase step)
        cuda_check(cudaMemcpyAsync(host_grad[static_cast<size_t>(l % host_grad_ring)], g, 4 * loc_now,
                                   cudaMemcpyDeviceToHost, s_d2h),
                   "grad");
        if (loc_late > 0)
          cuda_check(cudaMemcpyAsync(host_retain[static_cast<size_t>(l)], g + loc_now, 4 * loc_late,
                                     cudaMemcpyDeviceToHost, s_d2h),
                     "grad");
        if (t.bytes > 4 * n_my)  // shard padding (never with equal shards)
          cuda_check(cudaMemcpyAsync(host_grad[static_cast<size_t>(l % host_grad_ring)] + 4 * n_my, g + n_my,
                                     t.bytes - 4 * n_my, cudaMemcpyDeviceToHost, s_d2h),
                     "grad");
      } else if (t.link == LinkKind::PCIe_D2H) {
        cuda_check(cudaMemcpyAsync(host_grad[static_cast<size_t>(l % host_grad_ring)], g, t.bytes,
                                   cudaMemcpyDeviceToHost, s_d2h),
                   "grad");
      } else {
        cuda_check(cudaMemcpyAsync(g, host_grad[static_cast<size_t>(l % host_grad_ring)], t.bytes,
                                   cudaMemcpyHostToDevice, s_h2d),
                   "grad");
      }
      phys = t.bytes;
      break;
    }
    case DataKind::InterlayerGrad: {
      if (t.link == LinkKind::PCIe_D2H) {
        cuda_check(cudaMemcpyAsync(host_ilg[static_cast<size_t>(par * M + m)], ck(out_g, par, m), cb,
                                   cudaMemcpyDeviceToHost, s_d2h),
                   "ilg");
      } else {
        cuda_check(cudaMemcpyAsync(ck(in_g, par, m), host_ilg[static_cast<size_t>(parm1 * M + m)], cb,
                                   cudaMemcpyHostToDevice, s_h2d),
                   "ilg");
      }
      phys = cb;
      break;
    }
    case DataKind::OptState: {
      Blob& b = opt_blob[static_cast<size_t>(l)];
      const bool late = delayed(t) && !horizontal;
      const u64 lo = late ? 12 * loc_now : 0, hi = late ? b.size : 12 * loc_now;
      phys = ssd_io(b, lo, hi, t.link == LinkKind::SSD_Write);
      break;
    }
  }
}

void Executor::Impl::dispatch(Resource r, int iterations) {
  try {
    cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
    const auto& q = queue[static_cast<size_t>(r)];
    for (int it = 0; it < iterations; ++it) {
      // at most three iterations in flight (event slots are it % 3)
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] {
          if (failed.load()) return true;
          for (const auto& f : finished)
            if (f.load() < it - 2) return false;
          return true;
        });
      }
      if (failed.load()) return;
      for (int id : q) run_task(id, it);
      {
        std::lock_guard<std::mutex> g(mu);
        finished[static_cast<size_t>(r)].store(it);
      }
      cv.notify_all();
    }
  } catch (const std::exception& e) {
    {
      std::lock_guard<std::mutex> g(mu);
      if (!failed.load()) error = e.what();
      failed.store(true);
    }
    cv.notify_all();
  }
}

// =========================================================================
Executor::Executor(const SchedulePlan& plan, const ExecConfig& cfg) : impl_(std::make_unique<Impl>(plan, cfg)) {}
Executor::~Executor() = default;
const SchedulePlan& Executor::plan() const { return impl_->plan; }
const ExecConfig& Executor::config() const { return impl_->cfg; }

ExecReport Executor::run(int iterations, const int32_t* tokens, bool tokens_on_device) {
  Impl& I = *impl_;
  if (iterations < 1) throw ValidationError("run: iterations must be >= 1");
  if (!tokens) throw ValidationError("run: tokens required");
  const long long tok_n = 1LL * I.M * I.d.b * (I.d.s + 1);
  if (!tokens_on_device) {
    // ids index wte / dwte: reject out-of-vocabulary ids before any copy
    const long long n = tok_n * iterations;
    for (long long i = 0; i < n; ++i)
      if (tokens[i] < 0 || tokens[i] >= I.d.V)
        throw ValidationError("run: token id " + std::to_string(tokens[i]) + " at index " + std::to_string(i) +
                              " is outside [0, vocab_size)");
    if (I.tok_capacity < tok_n * iterations) {
      I.tok_pinned = reinterpret_cast<int32_t*>(I.arena.alloc(4ull * tok_n * iterations));
      I.tok_capacity = tok_n * iterations;
    }
    std::memcpy(I.tok_pinned, tokens, 4ull * tok_n * iterations);
    I.run_tokens = I.tok_pinned;
  } else {
    I.run_tokens = tokens;
  }
  I.run_tokens_dev = tokens_on_device;
  if (I.loss_cap < iterations) {
    I.dev_loss = static_cast<double*>(I.dmalloc(sizeof(double) * static_cast<u64>(iterations)));
    I.loss_cap = iterations;
  }
  for (auto& f : I.finished) f.store(-1);
  for (auto& di : I.done_iter) di.store(-1);
  I.failed.store(false);
  I.error.clear();
  I.led_logical = TrafficLedger{};
  I.led_ext = TrafficLedger{};
  I.led_phys = TrafficLedger{};
  I.last_iter = iterations - 1;
  I.trace.clear();
  I.launches.store(0);
  {
    const char* e = getenv("GS_HOST_PROF");
    I.host_prof = e && atoi(e) != 0;
    I.host_wait_s = I.host_enqueue_s = 0.0;
  }
  I.prof.reset();

  cuda_check(cudaDeviceSynchronize(), "pre-run sync");
  cuda_check(cudaEventRecord(I.ev_base, I.s_gpu), "base");
  cuda_check(cudaEventSynchronize(I.ev_base), "base");
  I.host_base = std::chrono::steady_clock::now();
  // H2D/D2H/opt streams start after the base event
  for (cudaStream_t s : {I.s_h2d, I.s_d2h, I.s_opt}) cuda_check(cudaStreamWaitEvent(s, I.ev_base, 0), "base wait");

  std::vector<std::thread> ts;
  for (int r = 0; r < kNumResources; ++r)
    ts.emplace_back([&I, r, iterations] { I.dispatch(static_cast<Resource>(r), iterations); });
  for (auto& t : ts) t.join();
  if (I.failed.load()) {
    cudaDeviceSynchronize();
    throw std::runtime_error("executor run failed: " + I.error);
  }
  // join all streams, then stop the clock
  cudaEvent_t ev_end;
  cuda_check(cudaEventCreate(&ev_end), "event");
  for (cudaStream_t s : {I.s_h2d, I.s_d2h, I.s_opt}) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(e, s), "record");
    cuda_check(cudaStreamWaitEvent(I.s_gpu, e, 0), "join");
    cudaEventDestroy(e);
  }
  std::vector<double> loss(static_cast<size_t>(iterations));
  ExecReport rep;
  cuda_check(cudaEventRecord(ev_end, I.s_gpu), "record");
  cuda_check(cudaEventSynchronize(ev_end), "sync");
  float ms = 0.0f;
  cuda_check(cudaEventElapsedTime(&ms, I.ev_base, ev_end), "elapsed");
  rep.total_ms = ms;
  if (I.host_prof)
    fprintf(stderr, "[gs host] %d iterations: GPU %.1f ms, compute dispatcher enqueue %.1f ms, dep waits %.1f ms\n",
            iterations, ms, 1e3 * I.host_enqueue_s, 1e3 * I.host_wait_s);
  cuda_check(cudaMemcpy(loss.data(), I.dev_loss, sizeof(double) * loss.size(), cudaMemcpyDeviceToHost), "loss");
  cudaEventDestroy(ev_end);
  int bad = 0;
  cuda_check(cudaMemcpy(&bad, I.dev_bad_tokens, sizeof(int), cudaMemcpyDeviceToHost), "token check");
  if (bad) {
    cuda_check(cudaMemset(I.dev_bad_tokens, 0, sizeof(int)), "memset");
    throw ValidationError("run: " + std::to_string(bad) +
                          " device token ids were outside [0, vocab_size) (replaced by 0; the run is invalid)");
  }
  const double denom = static_cast<double>(I.d.T()) * I.M;
  for (int it = 0; it < iterations; ++it) rep.losses.push_back(loss[static_cast<size_t>(it)] / denom);
  if (I.cfg.record_trace) {
    // CUDA events are recycled every 3 iterations: keep the last three
    std::vector<TraceRecord> kept;
    for (const TraceRecord& rec : I.trace)
      if (rec.iteration >= iterations - 3) kept.push_back(rec);
    I.trace.swap(kept);
    for (TraceRecord& rec : I.trace) {
      if (!I.is_stream[static_cast<size_t>(rec.task)]) continue;
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, I.ev_base, I.ev_start[static_cast<size_t>(rec.task)][static_cast<size_t>(rec.iteration % 3)]);
      cudaEventElapsedTime(&b, I.ev_base, I.ev_done[static_cast<size_t>(rec.task)][static_cast<size_t>(rec.iteration % 3)]);
      rec.t_start_ms = a;
      rec.t_end_ms = b;
    }
    rep.trace = I.trace;
  }
  I.global_iter += iterations;
  rep.ledger = I.led_logical;
  rep.extension = I.led_ext;
  rep.physical = I.led_phys;
  rep.gpu_bytes_allocated = I.dev_bytes;
  rep.host_pinned_bytes = I.arena.bytes();
  rep.gpu_launches = I.launches.load();
  return rep;
}

void Executor::flush() {
  Impl& I = *impl_;
  cuda_check(cudaDeviceSynchronize(), "flush sync");
  const u64 lp = static_cast<u64>(I.d.lp());
  for (int l = 0; l < I.N; ++l) {
    const long long ready = I.late_ready[static_cast<size_t>(l)].load();
    if (I.el_late == 0 || ready < 0 || I.late_applied[static_cast<size_t>(l)].load() >= ready) continue;
    if (I.loc_late > 0) {
      Blob& ob = I.opt_blob[static_cast<size_t>(l)];
      Blob& pb = I.param_blob[static_cast<size_t>(l)];
      // SSD-resident state: file -> staging slot, step, staging -> file
      if (I.ssd_opt) I.ssd_io(ob, 12 * I.loc_now, ob.size, false);
      if (I.host_step) {
        I.apply_adam_host(l, I.loc_now, I.n_my, I.host_retain[static_cast<size_t>(l)], static_cast<int>(ready + 1));
      } else {
        I.apply_adam(l, I.loc_now, I.n_my, I.retain[static_cast<size_t>(l)], static_cast<int>(ready + 1), I.s_opt, -2,
                     Src::Image);
        cuda_check(cudaStreamSynchronize(I.s_opt), "flush step");
      }
      if (I.ssd_opt) I.ssd_io(ob, 12 * I.loc_now, ob.size, true);
      if (I.ssd_param) I.ssd_io(pb, lp * I.loc_now, pb.size, true);
    }
    I.late_applied[static_cast<size_t>(l)].store(ready);
  }
  if (I.fixed_done < I.global_iter) {
    if (I.dp) I.fixed_allreduce(I.s_opt);
    gs::AdamHyper hp{I.cfg.adam.lr, I.cfg.adam.beta1, I.cfg.adam.beta2, I.cfg.adam.eps, I.cfg.adam.weight_decay};
    cuda_check(gs::adam_step(hp, static_cast<int>(I.global_iter), 1.0f, I.fx_master, I.fx_m, I.fx_v, I.fx_grad, I.fx_lp,
                             I.d.dt, I.n_fixed, I.s_opt),
               "fixed adam");
    cuda_check(cudaMemsetAsync(I.fx_grad, 0, 4 * I.n_fixed, I.s_opt), "fixed grad");
    I.fixed_done = I.global_iter;
  }
  cuda_check(cudaDeviceSynchronize(), "flush sync");
}

namespace {
// Reads field `f` (0 master, 1 m, 2 v) of every element of an opt blob.
void read_field(Executor::Impl& I, int layer, int f, float* out);
}  // namespace

void Executor::read_params(float* layers, float* fixed) {
  Impl& I = *impl_;
  cuda_check(cudaDeviceSynchronize(), "sync");
  if (layers)
    for (int l = 0; l < I.N; ++l) read_field(I, l, 0, layers + static_cast<size_t>(l) * I.P);
  if (fixed) cuda_check(cudaMemcpy(fixed, I.fx_master, 4 * I.n_fixed, cudaMemcpyDeviceToHost), "read fixed");
}

void Executor::read_moments(float* layer_m, float* layer_v, float* fixed_m, float* fixed_v) {
  Impl& I = *impl_;
  cuda_check(cudaDeviceSynchronize(), "sync");
  for (int l = 0; l < I.N; ++l) {
    if (layer_m) read_field(I, l, 1, layer_m + static_cast<size_t>(l) * I.P);
    if (layer_v) read_field(I, l, 2, layer_v + static_cast<size_t>(l) * I.P);
  }
  if (fixed_m) cuda_check(cudaMemcpy(fixed_m, I.fx_m, 4 * I.n_fixed, cudaMemcpyDeviceToHost), "read fixed m");
  if (fixed_v) cuda_check(cudaMemcpy(fixed_v, I.fx_v, 4 * I.n_fixed, cudaMemcpyDeviceToHost), "read fixed v");
}

namespace {
void read_field(Executor::Impl& I, int layer, int f, float* out) {
  const Blob& b = I.opt_blob[static_cast<size_t>(layer)];
  std::vector<uint8_t> all(b.size);
  for (const Segment& s : b.segs) {
    if (s.tier == Tier::Hbm) {
      cuda_check(cudaMemcpy(all.data() + s.lo, s.dev, s.size(), cudaMemcpyDeviceToHost), "read opt");
    } else if (s.tier == Tier::Dram) {
      std::memcpy(all.data() + s.lo, s.img, s.size());
    } else {  // the NVMe file holds the only copy
      const u64 n = align_up(s.size(), kNvmeAlign);
      void* tmp = nullptr;
      if (posix_memalign(&tmp, kNvmeAlign, n) != 0) throw std::bad_alloc();
      I.nvme->read(s.file_off, tmp, s.size());
      std::memcpy(all.data() + s.lo, tmp, s.size());
      std::free(tmp);
    }
  }
  const float* st = reinterpret_cast<const float*>(all.data());
  // this rank's shard [e_lo, e_hi) of the layer (the whole layer when W == 1)
  for (u64 i = 0; i < I.n_my; ++i) out[I.e_lo + i] = st[3 * i + static_cast<u64>(f)];
}
}  // namespace

Executor::KernelTotals Executor::kernel_profile() const {
  KernelTotals t{};
  impl_->prof.totals(t.flops, t.ms, t.launches, t.total);
  impl_->prof.span_totals(&t.span_flops, &t.span_ms, &t.span_launches);
  if (const char* p = getenv("GS_PROF_DUMP")) impl_->prof.dump_pairs(p);
  return t;
}

void Executor::set_trace(bool on) {
  Impl& I = *impl_;
  cuda_check(cudaDeviceSynchronize(), "sync");
  if (on && I.ev_start.empty()) {
    const size_t n = I.plan.tasks.size();
    I.ev_start.resize(n);
    for (size_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) {
        I.ev_start[i][static_cast<size_t>(k)] = nullptr;
        if (!I.is_stream[i]) continue;
        cudaEventDestroy(I.ev_done[i][static_cast<size_t>(k)]);  // timing-enabled replacements
        cuda_check(cudaEventCreate(&I.ev_done[i][static_cast<size_t>(k)]), "event");
        cuda_check(cudaEventCreate(&I.ev_start[i][static_cast<size_t>(k)]), "event");
      }
  }
  I.cfg.record_trace = on;
}

void Executor::set_profiling(int stride) {
  impl_->prof.stride = stride > 0 ? stride : 1;
  impl_->ws.prof = stride > 0 ? &impl_->prof : nullptr;
}

ExecReport execute(const SchedulePlan& plan, const ExecConfig& cfg, int iterations, const int32_t* tokens) {
  Executor ex(plan, cfg);
  return ex.run(iterations, tokens);
}

}  // namespace offsim
