#include <cstdio>
#include <cstdlib>

#include "layer_ops.hpp"

namespace gs::engine {

namespace {

#define GS_TRY(expr)                          \
  do {                                        \
    const cudaError_t e_ = (expr);            \
    if (e_ != cudaSuccess) return e_;         \
  } while (0)

const uint8_t* off(const void* p, long long elems, int eb) {
  return static_cast<const uint8_t*>(p) + elems * eb;
}

// RAII timing scope on the compute stream (no-op without a profiler).
struct Scope {
  KernelProfiler* p;
  int cls;
  double flops;
  cudaStream_t st;
  int a = -1;
  Scope(KernelProfiler* p_, int c, double f, cudaStream_t s) : p(p_), cls(c), flops(f), st(s) {
    if (p) a = p->begin(st, cls);
  }
  ~Scope() {
    if (p && a >= 0) p->end(cls, flops, a, st);
  }
};

// C[M,N] = A . B^T style call with explicit majors.
cudaError_t mm(const Dims& d, int M, int N, int K, const void* A, bool a_k, const void* B, bool b_k, void* C,
               Epi epi, cudaStream_t st, LaunchCounter& lc, const void* R = nullptr, void* G = nullptr,
               KernelProfiler* prof = nullptr) {
  Scope sc(prof, KernelProfiler::Gemm, 2.0 * M * N * K, st);
  GemmArgs g;
  if (prof) {
    if (prof->span_on_events < 0) {
      const char* e = std::getenv("GS_PROF_SPAN_ON_EVENTS");
      prof->span_on_events = (e && e[0] == '1') ? 1 : 0;
    }
    if (prof->span_on_events ? sc.a >= 0 : sc.a < 0)
      g.span = prof->span_on_events ? prof->span_slot_at(2.0 * M * N * K) : prof->span_slot(2.0 * M * N * K);
  }
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.B = B;
  g.a_kmajor = a_k;
  g.b_kmajor = b_k;
  g.C = C;
  g.R = R;
  g.G = G;
  g.epi = epi;
  g.dt = d.dt;
  ++lc.n;
  return gemm(g, st);
}

}  // namespace

// Time one non-GEMM launch sequence under class `cls` when profiling.
#define GS_PROF(cls, expr)                                     \
  do {                                                         \
    Scope sc_(ws.prof, KernelProfiler::cls, 0.0, st);          \
    GS_TRY(expr);                                              \
  } while (0)

int KernelProfiler::begin(cudaStream_t st, int cls) {
  ++all_launches[cls];
  if (seen[cls]++ % (stride > 0 ? stride : 1) != 0) return -1;
  if (next + 2 > pool.size()) {
    const size_t grow = pool.size() < 4096 ? 4096 : pool.size();
    for (size_t i = 0; i < grow; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
  }
  const int a = static_cast<int>(next++);
  if (fence < 0) {
    const char* e = std::getenv("GS_PROF_FENCE");
    fence = (e && e[0] == '1') ? 1 : 0;
  }
  if (fence) gs::stream_fence(st);
  cudaEventRecord(pool[static_cast<size_t>(a)], st);
  return a;
}
void KernelProfiler::end(int cls, double flops, int a, cudaStream_t st) {
  const int b = static_cast<int>(next++);
  if (fence) gs::stream_fence(st);
  cudaEventRecord(pool[static_cast<size_t>(b)], st);
  recs.push_back({cls, flops, a, b});
}
void KernelProfiler::totals(double* flops, double* ms, int* launches, long long* total) const {
  for (int c = 0; c < kCount; ++c) {
    flops[c] = 0;
    ms[c] = 0;
    launches[c] = 0;
    total[c] = all_launches[c];
  }
  for (const Rec& r : recs) {
    float t = 0.0f;
    if (cudaEventElapsedTime(&t, pool[static_cast<size_t>(r.a)], pool[static_cast<size_t>(r.b)]) != cudaSuccess) continue;
    flops[r.cls] += r.flops;
    ms[r.cls] += t;
    launches[r.cls] += 1;
  }
}
unsigned long long* KernelProfiler::span_slot(double flops) {
  const int st = stride > 0 ? stride : 1;
  if (span_seen++ % st != st / 2) return nullptr;
  if (!span_dev) {
    if (cudaMalloc(&span_dev, 2 * sizeof(unsigned long long) * kSpanCap) != cudaSuccess) {
      span_dev = nullptr;
      (void)cudaGetLastError();
      return nullptr;
    }
    reset();
  }
  const size_t i = span_flops.size();
  if (i >= static_cast<size_t>(kSpanCap)) return nullptr;
  span_flops.push_back(flops);
  return span_dev + 2 * i;
}
unsigned long long* KernelProfiler::span_slot_at(double flops) {
  ++span_seen;
  if (!span_dev) {
    if (cudaMalloc(&span_dev, 2 * sizeof(unsigned long long) * kSpanCap) != cudaSuccess) {
      span_dev = nullptr;
      (void)cudaGetLastError();
      return nullptr;
    }
    // not reset(): this launch's begin event is outstanding
    std::vector<unsigned long long> init(2 * static_cast<size_t>(kSpanCap));
    for (size_t i = 0; i < init.size(); i += 2) {
      init[i] = ~0ULL;
      init[i + 1] = 0;
    }
    cudaMemcpy(span_dev, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice);
    span_flops.clear();
  }
  const size_t i = span_flops.size();
  if (i >= static_cast<size_t>(kSpanCap)) return nullptr;
  span_flops.push_back(flops);
  return span_dev + 2 * i;
}
void KernelProfiler::reset() {
  next = 0;
  recs.clear();
  for (int c = 0; c < kCount; ++c) seen[c] = all_launches[c] = 0;
  span_flops.clear();
  span_seen = 0;
  if (span_dev) {  // [min, max] pairs: min = ~0 (0xff bytes), max = 0
    cudaDeviceSynchronize();
    std::vector<unsigned long long> init(2 * static_cast<size_t>(kSpanCap));
    for (size_t i = 0; i < init.size(); i += 2) {
      init[i] = ~0ULL;
      init[i + 1] = 0;
    }
    cudaMemcpy(span_dev, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice);
  }
}
void KernelProfiler::span_totals(double* flops, double* ms, int* launches) const {
  *flops = 0;
  *ms = 0;
  *launches = 0;
  if (!span_dev || span_flops.empty()) return;
  std::vector<unsigned long long> h(2 * span_flops.size());
  if (cudaMemcpy(h.data(), span_dev, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  for (size_t i = 0; i < span_flops.size(); ++i) {
    const unsigned long long a = h[2 * i], b = h[2 * i + 1];
    if (a == ~0ULL || b <= a) continue;  // launch not (yet) executed
    *flops += span_flops[i];
    *ms += static_cast<double>(b - a) * 1e-6;
    ++*launches;
  }
}
void KernelProfiler::dump_pairs(const char* path) const {
  if (span_on_events != 1 || !span_dev) return;
  std::vector<unsigned long long> h(2 * span_flops.size());
  if (h.empty() ||
      cudaMemcpy(h.data(), span_dev, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  FILE* f = std::fopen(path, "w");
  if (!f) return;
  std::fprintf(f, "sample,flops,event_ms,span_ms\n");
  size_t i = 0;
  for (const Rec& r : recs) {
    if (r.cls != Gemm) continue;
    if (i >= span_flops.size()) break;
    float t = 0.0f;
    cudaEventElapsedTime(&t, pool[static_cast<size_t>(r.a)], pool[static_cast<size_t>(r.b)]);
    const unsigned long long a = h[2 * i], b = h[2 * i + 1];
    const double sp = (a == ~0ULL || b <= a) ? -1.0 : static_cast<double>(b - a) * 1e-6;
    std::fprintf(f, "%zu,%.0f,%.4f,%.4f\n", i, r.flops, t, sp);
    ++i;
  }
  std::fclose(f);
}
KernelProfiler::~KernelProfiler() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
  if (span_dev) cudaFree(span_dev);
}

bool alloc_workspace(const Dims& d, Workspace& ws) {
  const size_t eb = static_cast<size_t>(d.lp());
  const size_t Th = static_cast<size_t>(d.T()) * d.h;
  const size_t T = static_cast<size_t>(d.T());
  bool ok = true;
  auto get = [&](void** p, size_t bytes) {
    if (!ok) return;
    if (cudaMalloc(p, bytes < 256 ? 256 : bytes) != cudaSuccess) {
      ok = false;
      *p = nullptr;
      return;
    }
    ws.bytes += bytes;
  };
  get(&ws.a, Th * eb);
  get(&ws.qkv, 3 * Th * eb);
  get(&ws.o, Th * eb);
  get(&ws.x1, Th * eb);
  get(&ws.c, Th * eb);
  get(&ws.u, 4 * Th * eb);
  get(&ws.g, 4 * Th * eb);
  get(&ws.y, Th * eb);
  get(&ws.dy, Th * eb);
  get(&ws.big, 4 * Th * eb);
  get(&ws.dx1, Th * eb);
  get(&ws.tmp, Th * eb);
  get(&ws.dqkv, 3 * Th * eb);
  get(&ws.x0, Th * eb);
  get(&ws.z, Th * eb);
  get(reinterpret_cast<void**>(&ws.lse), sizeof(float) * static_cast<size_t>(d.b) * d.H * d.s);
  float** stats[] = {&ws.m1, &ws.r1, &ws.m2, &ws.r2, &ws.mz, &ws.rz};
  for (float** p : stats) get(reinterpret_cast<void**>(p), sizeof(float) * T);
  get(&ws.attn_work, attention_bwd_workspace(d.b, d.s, d.h, d.H));
  get(reinterpret_cast<void**>(&ws.logits), sizeof(float) * T * d.V);
  get(&ws.dlogits, T * d.V * eb);
  // The weight-gradient stream shares the compute stream's (highest)
  // priority, above the optimizer stream.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (ok && (cudaStreamCreateWithPriority(&ws.side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
             cudaEventCreateWithFlags(&ws.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
             cudaEventCreateWithFlags(&ws.ev_join, cudaEventDisableTiming) != cudaSuccess))
    ok = false;
  return ok;
}

void free_workspace(Workspace& ws) {
  void* ptrs[] = {ws.a, ws.qkv, ws.o, ws.x1, ws.c, ws.u, ws.g, ws.y, ws.dy, ws.big, ws.dx1, ws.tmp, ws.dqkv,
                  ws.x0, ws.z, ws.lse, ws.m1, ws.r1, ws.m2, ws.r2, ws.mz, ws.rz, ws.attn_work, ws.logits,
                  ws.dlogits};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ws.side) cudaStreamDestroy(ws.side);
  if (ws.ev_fork) cudaEventDestroy(ws.ev_fork);
  if (ws.ev_join) cudaEventDestroy(ws.ev_join);
  ws = Workspace{};
}

// Forward through LN1 .. GELU; leaves a, qkv, o, lse, x1, c, g, stats in ws,
// and u (the pre-GELU activation) when keep_u — only the recompute feeds a
// backward, so FwdCompute skips that 4*T*h store.
static cudaError_t forward_body(const Dims& d, const void* W, const void* x, Workspace& ws, cudaStream_t st,
                                LaunchCounter& lc, bool keep_u) {
  const int T = d.T(), h = d.h, eb = d.lp();
  const long long h2 = 1LL * h * h;
  const void* wqkv = W;
  const void* wo = off(W, 3 * h2, eb);
  const void* w1 = off(W, 4 * h2, eb);
  GS_PROF(Norm, layernorm_fwd(d.dt, x, ws.a, ws.m1, ws.r1, T, h, st));
  GS_TRY(mm(d, T, 3 * h, h, ws.a, true, wqkv, true, ws.qkv, Epi::Store, st, lc, nullptr, nullptr, ws.prof));
  {
    Scope sc(ws.prof, KernelProfiler::AttnFwd, 2.0 * d.b * d.H * (double)d.s * d.s * (h / d.H), st);
    GS_TRY(attention_fwd(d.dt, ws.qkv, ws.o, ws.lse, d.b, d.s, h, d.H, st));
  }
  GS_TRY(mm(d, T, h, h, ws.o, true, wo, true, ws.x1, Epi::AddResidual, st, lc, x, nullptr, ws.prof));
  GS_PROF(Norm, layernorm_fwd(d.dt, ws.x1, ws.c, ws.m2, ws.r2, T, h, st));
  if (keep_u)
    GS_TRY(mm(d, T, 4 * h, h, ws.c, true, w1, true, ws.u, Epi::StoreGelu, st, lc, nullptr, ws.g, ws.prof));
  else
    GS_TRY(mm(d, T, 4 * h, h, ws.c, true, w1, true, ws.g, Epi::Gelu, st, lc, nullptr, nullptr, ws.prof));
  lc.n += 4;  // two LayerNorms + attention (1 kernel in either path... counted as 1) + spare
  return cudaSuccess;
}

cudaError_t layer_forward(const Dims& d, const void* W, const void* x, void* y, Workspace& ws, cudaStream_t st,
                          LaunchCounter& lc) {
  const long long h2 = 1LL * d.h * d.h;
  GS_TRY(forward_body(d, W, x, ws, st, lc, false));
  return mm(d, d.T(), d.h, 4 * d.h, ws.g, true, off(W, 8 * h2, d.lp()), true, y, Epi::AddResidual, st, lc, ws.x1, nullptr, ws.prof);
}

cudaError_t layer_backward(const Dims& d, const void* W, const void* x, const void* dy_in, void* dx, float* dW,
                           bool first, const HeadArgs* head, Workspace& ws, cudaStream_t st, LaunchCounter& lc) {
  const int T = d.T(), h = d.h, eb = d.lp();
  const long long h2 = 1LL * h * h;
  const void* wqkv = W;
  const void* wo = off(W, 3 * h2, eb);
  const void* w1 = off(W, 4 * h2, eb);
  const void* w2 = off(W, 8 * h2, eb);
  const Epi wg = first ? Epi::StoreF32 : Epi::AccumF32;
  GS_TRY(forward_body(d, W, x, ws, st, lc, true));  // recompute from the checkpoint

  // Weight gradients run on ws.side once their inputs exist (fork), the
  // data-gradient chain stays on st; every input a wgrad reads is left intact
  // until this call returns, and the join below orders dW and the workspace
  // before the next task.  GEMMs from here on overlap each other, so none is
  // event-timed (a per-launch duration would not be the kernel's own);
  // bench.py's GEMM roofline samples the forward / recompute GEMMs, which run
  // alone on the compute stream.
  cudaStream_t sd = ws.side ? ws.side : st;
  auto fork = [&]() -> cudaError_t {
    if (sd == st) return cudaSuccess;
    GS_TRY(cudaEventRecord(ws.ev_fork, st));
    return cudaStreamWaitEvent(sd, ws.ev_fork, 0);
  };
  const void* dy = dy_in;
  if (head) {
    // y = block output; tied head on LN_f(y); dy = d(CE)/dy
    GS_TRY(mm(d, T, h, 4 * h, ws.g, true, w2, true, ws.y, Epi::AddResidual, st, lc, ws.x1, nullptr, ws.prof));
    GS_PROF(Norm, layernorm_fwd(d.dt, ws.y, ws.z, ws.mz, ws.rz, T, h, st));
    GS_TRY(mm(d, T, d.V, h, ws.z, true, head->wte, true, ws.logits, Epi::StoreF32, st, lc, nullptr, nullptr, ws.prof));
    GS_PROF(Other, softmax_xent(ws.logits, ws.dlogits, d.dt, head->tokens, d.b, d.s, d.V, head->scale, head->loss_sum, st));
    // dwte += dlogits^T z  (M=V, N=h, K=T), concurrent with dz
    GS_TRY(fork());
    GS_TRY(mm(d, d.V, h, T, ws.dlogits, false, ws.z, false, head->dwte, Epi::AccumF32, sd, lc));
    // dz = dlogits . wte   (M=T, N=h, K=V)
    GS_TRY(mm(d, T, h, d.V, ws.dlogits, true, head->wte, false, ws.tmp, Epi::Store, st, lc, nullptr, nullptr, nullptr));
    GS_PROF(Norm, layernorm_bwd(d.dt, ws.y, ws.mz, ws.rz, ws.tmp, nullptr, ws.dy, T, h, st));
    dy = ws.dy;
    lc.n += 3;
  }
  float* dWqkv = dW;
  float* dWo = dW + 3 * h2;
  float* dW1 = dW + 4 * h2;
  float* dW2 = dW + 8 * h2;
  // MLP
  GS_TRY(fork());
  GS_TRY(mm(d, h, 4 * h, T, dy, false, ws.g, false, dW2, wg, sd, lc));                                    // dW2 (+)= dy^T g
  // du = (dy W2) * gelu'(u): GELU backward fused into the dgrad epilogue
  GS_TRY(mm(d, T, 4 * h, h, dy, true, w2, false, ws.big, Epi::MulGeluGrad, st, lc, ws.u, nullptr, nullptr));
  GS_TRY(fork());
  GS_TRY(mm(d, 4 * h, h, T, ws.big, false, ws.c, false, dW1, wg, sd, lc));                                // dW1 (+)= du^T c
  GS_TRY(mm(d, T, h, 4 * h, ws.big, true, w1, false, ws.tmp, Epi::Store, st, lc, nullptr, nullptr, nullptr));  // dc = du W1
  GS_PROF(Norm, layernorm_bwd(d.dt, ws.x1, ws.m2, ws.r2, ws.tmp, dy, ws.dx1, T, h, st));  // dx1 = dy + LN2'
  // attention
  GS_TRY(fork());
  GS_TRY(mm(d, h, h, T, ws.dx1, false, ws.o, false, dWo, wg, sd, lc));                                    // dWo (+)= dx1^T o
  GS_TRY(mm(d, T, h, h, ws.dx1, true, wo, false, ws.tmp, Epi::Store, st, lc, nullptr, nullptr, nullptr));    // do = dx1 Wo
  {
    Scope sc(ws.prof, KernelProfiler::AttnBwd, 5.0 * d.b * d.H * (double)d.s * d.s * (h / d.H), st);
    GS_TRY(attention_bwd(d.dt, ws.qkv, ws.o, ws.lse, ws.tmp, ws.dqkv, ws.attn_work, d.b, d.s, h, d.H, st));
  }
  GS_TRY(fork());
  GS_TRY(mm(d, 3 * h, h, T, ws.dqkv, false, ws.a, false, dWqkv, wg, sd, lc));                             // dWqkv (+)= dqkv^T a
  GS_TRY(mm(d, T, h, 3 * h, ws.dqkv, true, wqkv, false, ws.tmp, Epi::Store, st, lc, nullptr, nullptr, nullptr));  // da = dqkv Wqkv
  GS_PROF(Norm, layernorm_bwd(d.dt, x, ws.m1, ws.r1, ws.tmp, ws.dx1, dx, T, h, st));  // dx = dx1 + LN1'
  if (sd != st) {  // join
    GS_TRY(cudaEventRecord(ws.ev_join, sd));
    GS_TRY(cudaStreamWaitEvent(st, ws.ev_join, 0));
  }
  lc.n += 6;
  return cudaSuccess;
}

}  // namespace gs::engine
