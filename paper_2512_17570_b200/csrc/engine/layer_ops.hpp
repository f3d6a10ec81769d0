// GPU work of the plan's compute tasks (FwdCompute, RecomputeAndBwd and the
// head / embedding parts of FixedOps), one micro-batch at a time.  The math
// is the oracle's (oracle/gs_oracle.c): pre-LN GPT block with exactly 12h^2
// parameters laid out [Wqkv 3h^2 | Wo h^2 | W1 4h^2 | W2 4h^2], each [out][in].
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kernels.h"

namespace gs::engine {

struct Dims {
  int b = 1, s = 1, h = 1, H = 1, V = 1;
  DType dt = DType::BF16;
  int T() const { return b * s; }
  int lp() const { return dtype_bytes(dt); }
  long long P() const { return 12LL * h * h; }
};

// Optional per-kernel-class CUDA-event timing of the compute stream
// (bench.py's live roofline numbers).  Classes: see kProfClasses.
struct KernelProfiler {
  enum Cls { Gemm = 0, AttnFwd, AttnBwd, Norm, Other, kCount };
  struct Rec {
    int cls;
    double flops;
    int a, b;  // indices into pool
  };
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<Rec> recs;
  // Time one launch in `stride` per class (an event pair between back-to-back
  // persistent kernels costs a pipeline drain); totals are ratio estimates.
  int stride = 16;
  long long seen[kCount] = {};
  long long all_launches[kCount] = {};
  int begin(cudaStream_t st, int cls);           // event index, or -1 when not sampled
  void end(int cls, double flops, int a, cudaStream_t st);
  // In-kernel span samples of the tcgen05 GEMM (GemmArgs::span): one launch
  // in `stride`, offset stride / 2 from the event-timed ones, records its
  // first-CTA-start .. last-CTA-exit %globaltimer span.  No stream operation
  // sits between the kernels, so programmatic dependent launch and the
  // step's timing are undisturbed (an event pair costs each timed launch its
  // launch ramp).  Device buffer: [kSpanCap] minima, then [kSpanCap] maxima.
  static constexpr int kSpanCap = 1 << 15;
  unsigned long long* span_dev = nullptr;
  std::vector<double> span_flops;
  long long span_seen = 0;
  unsigned long long* span_slot(double flops);  // nullptr when not sampled
  // GS_PROF_SPAN_ON_EVENTS=1 (diagnostic): take the span samples on the
  // event-bracketed launches instead, to split an event-timed duration into
  // the kernel's own span and the ramp before it.
  int span_on_events = -1;
  // GS_PROF_FENCE=1 (diagnostic): a no-op non-PDL grid before each event of
  // a timed pair, so the events mark completions of the work before them
  int fence = -1;
  unsigned long long* span_slot_at(double flops);
  void reset();
  // per class after the stream has completed: sampled flops, sampled ms,
  // sampled launches, all launches
  void totals(double* flops, double* ms, int* launches, long long* total) const;
  // GEMM span samples after the stream has completed
  void span_totals(double* flops, double* ms, int* launches) const;
  // GS_PROF_SPAN_ON_EVENTS diagnostics: per sampled GEMM launch, flops,
  // event ms and in-kernel span ms, one CSV line each
  void dump_pairs(const char* path) const;
  ~KernelProfiler();
};
inline const char* const kProfClasses[] = {"gemm", "attention_fwd", "attention_bwd", "layernorm", "other"};

// Per-micro-batch device scratch (allocated once per engine).
struct Workspace {
  KernelProfiler* prof = nullptr;
  void *a = nullptr, *qkv = nullptr, *o = nullptr, *x1 = nullptr, *c = nullptr, *u = nullptr, *g = nullptr;
  void *y = nullptr, *dy = nullptr, *big = nullptr, *dx1 = nullptr, *tmp = nullptr, *dqkv = nullptr, *x0 = nullptr;
  float *lse = nullptr, *m1 = nullptr, *r1 = nullptr, *m2 = nullptr, *r2 = nullptr, *mz = nullptr, *rz = nullptr;
  void* attn_work = nullptr;
  float* logits = nullptr;
  void* dlogits = nullptr;
  void* z = nullptr;
  uint64_t bytes = 0;
  // Second compute stream for the weight-gradient GEMMs: they are off the
  // backward's critical path (dgrad -> LN' -> attention' -> ...), so they
  // run concurrently and fill the dgrad kernels' tail waves and the small
  // kernels in between; joined back before layer_backward returns.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// Allocates every buffer of `ws`; returns false on cudaMalloc failure.
bool alloc_workspace(const Dims& d, Workspace& ws);
void free_workspace(Workspace& ws);

// Launch accounting (kernels enqueued by this thread's engine work).
struct LaunchCounter {
  int n = 0;
};

// y = block(x).  x, y: [T][h] in dt.  W: 12h^2 in dt.
cudaError_t layer_forward(const Dims& d, const void* W, const void* x, void* y, Workspace& ws, cudaStream_t st,
                          LaunchCounter& lc);

// Recompute block(x) and back-propagate dy.  dx: [T][h] (may be ws-free
// memory distinct from dy).  dW: fp32 12h^2, overwritten when `first` else
// accumulated.  When `head` is set, dy is produced here from the tied LM head
// on the recomputed output (layer N-1): loss_sum += CE, dwte += head grad.
struct HeadArgs {
  const void* wte = nullptr;  // [V][h] dt
  float* dwte = nullptr;      // [V][h] fp32
  const int32_t* tokens = nullptr;  // [b][s+1]
  float scale = 1.0f;         // 1 / (T * M * dp)
  double* loss_sum = nullptr;
};
cudaError_t layer_backward(const Dims& d, const void* W, const void* x, const void* dy, void* dx, float* dW,
                           bool first, const HeadArgs* head, Workspace& ws, cudaStream_t st, LaunchCounter& lc);

}  // namespace gs::engine
