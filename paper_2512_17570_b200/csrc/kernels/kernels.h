// Internal C++ launch API of the sm_100a kernels (host side).  The engine and
// the C-ABI wrappers (capi/kernels_capi.cu) call these; all are asynchronous
// on the given stream and report launch errors through the return value.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gs {

enum class DType { F32 = 0, BF16 = 1 };
inline int dtype_bytes(DType t) { return t == DType::F32 ? 4 : 2; }

// ---------------------------------------------------------------- GEMM
// C[M,N] = sum_k A(m,k) B(n,k), fp32 accumulation.
//   a_kmajor: A stored [M][K] (else [K][M]);  b_kmajor: B stored [N][K] (else [K][N])
// Epilogues:
enum class Epi {
  Store = 0,        // C(dt) = acc
  AddResidual = 1,  // C(dt) = acc + R(dt)
  AccumF32 = 2,     // Cf32 += acc
  StoreGelu = 3,    // C(dt) = acc, G(dt) = gelu(acc)
  StoreF32 = 4,     // Cf32 = acc
  MulGeluGrad = 5,  // C(dt) = acc * gelu'(R(dt))   (dgrad of FC2 fused with GELU backward)
  Gelu = 6,         // C(dt) = gelu(acc)   (StoreGelu's G alone: FwdCompute keeps no u)
};
struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr;
  const void* B = nullptr;
  bool a_kmajor = true, b_kmajor = true;
  void* C = nullptr;        // dt, or fp32 for AccumF32 / StoreF32
  const void* R = nullptr;  // residual (AddResidual)
  void* G = nullptr;        // gelu output (StoreGelu)
  int ldc = 0;              // leading dim of C / R / G (0 -> N)
  Epi epi = Epi::Store;
  DType dt = DType::BF16;   // operand / output storage type
  // optional in-kernel span sample (tcgen05 path): [0] min over CTAs of the
  // %globaltimer at work start (after the PDL wait), [1] max at CTA exit;
  // the caller pre-sets [0] = ~0, [1] = 0
  unsigned long long* span = nullptr;
};
// Chooses the tcgen05 path (bf16, tile-aligned shapes) or the SIMT path.
cudaError_t gemm(const GemmArgs& g, cudaStream_t s);
cudaError_t gemm_simt(const GemmArgs& g, cudaStream_t s);
cudaError_t gemm_tc(const GemmArgs& g, cudaStream_t s);  // tcgen05 + TMA + TMEM
bool gemm_tc_supported(const GemmArgs& g);

// ----------------------------------------------------------- attention
// qkv [b*s][3h] (q|k|v column blocks, head j at columns j*d), o [b*s][h],
// lse [b][H][s] fp32 (natural-log units of the 1/sqrt(d)-scaled scores).
cudaError_t attention_fwd(DType dt, const void* qkv, void* o, float* lse, int b, int s, int h,
                          int H, cudaStream_t st);
// dqkv [b*s][3h] = grads; needs the forward's o and lse.  `work` must hold
// attention_bwd_workspace() bytes.
size_t attention_bwd_workspace(int b, int s, int h, int H);
// tcgen05 forward (head_dim 128, bf16, s % 128 == 0); GS_ATTN_TC=0 disables
bool attention_tc_supported(DType dt, int s, int h, int H);
cudaError_t attention_fwd_tc(const void* qkv, void* o, float* lse, int b, int s, int h, int H, cudaStream_t st);
cudaError_t attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* lse2, const float* D,
                             void* dqkv,
                             float* dq_acc, int b, int s, int h, int H, cudaStream_t st);
cudaError_t attention_bwd(DType dt, const void* qkv, const void* o, const float* lse, const void* dout,
                          void* dqkv, void* work, int b, int s, int h, int H, cudaStream_t st);

// ------------------------------------------------------- normalisation
// non-affine LayerNorm over rows of width h, eps = 1e-5
cudaError_t layernorm_fwd(DType dt, const void* x, void* y, float* mean, float* rstd, int rows, int h,
                          cudaStream_t s);
// dx = (res ? res : 0) + LN_backward(dy); res may alias dx (res = dx accumulates)
cudaError_t layernorm_bwd(DType dt, const void* x, const float* mean, const float* rstd, const void* dy,
                          const void* res, void* dx, int rows, int h, cudaStream_t s);

// ---------------------------------------------------------- elementwise
cudaError_t gelu_fwd(DType dt, const void* u, void* g, long long n, cudaStream_t s);
// du = dg * gelu'(u), in place on dg allowed
cudaError_t gelu_bwd(DType dt, const void* u, const void* dg, void* du, long long n, cudaStream_t s);
// y = a + b
cudaError_t add(DType dt, const void* a, const void* b, void* y, long long n, cudaStream_t s);
cudaError_t fill_zero(void* p, size_t bytes, cudaStream_t s);
// no-op grid without PDL: orders an event after its predecessor's completion
cudaError_t stream_fence(cudaStream_t s);
// dst[i] = src[i] by SM threads (src may be mapped pinned host memory): a
// small copy that does not queue behind bulk DMA on the copy engines.
cudaError_t copy_words(uint32_t* dst, const uint32_t* src, long long n, cudaStream_t s);
// dst[i] = src[i] for token ids, with ids outside [0, vocab) replaced by 0
// and counted into *bad (device int).
cudaError_t copy_tokens(int32_t* dst, const int32_t* src, long long n, int vocab, int* bad, cudaStream_t s);

// ----------------------------------------------------- embedding / head
// x0[bi*s+t] = wte[tok[bi*(s+1)+t]] + wpe[t]   (tokens laid out [b][s+1])
cudaError_t embed_fwd(DType dt, const void* wte, const void* wpe, const int32_t* tok, void* x0, int b,
                      int s, int h, cudaStream_t st);
// dwte[tok] += dx0, dwpe[t] += dx0 (fp32 grads, atomics)
cudaError_t embed_bwd(DType dt, const int32_t* tok, const void* dx0, float* dwte, float* dwpe, int b, int s,
                      int h, cudaStream_t st);
// In place: logits(fp32)[T][V] -> dlogits(dt) = (softmax - onehot) * scale,
// loss_sum[0] += sum_t CE_t (fp64 accumulator).  targets = tokens shifted.
cudaError_t softmax_xent(const float* logits, void* dlogits, DType dt, const int32_t* tok, int b, int s,
                         int V, float scale, double* loss_sum, cudaStream_t st);

// ------------------------------------------------------------ optimizer
struct AdamHyper {
  float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.0f;
};
// Fused Adam(W) over n elements: fp32 master/m/v updated in place from the
// fp32 gradient (x grad_scale), and the low-precision working copy written
// (param_lp may be null; lp_dt selects its type).  step is 1-based.
cudaError_t adam_step(const AdamHyper& hp, int step, float grad_scale, float* master, float* m, float* v,
                      const float* grad, void* param_lp, DType lp_dt, long long n, cudaStream_t s);
// Same update, optimizer state interleaved per element as [master, m, v]
// (12 bytes/elem), the layout of the offloaded opt-state blob.
cudaError_t adam_step_packed(const AdamHyper& hp, int step, float grad_scale, float* state,
                             const float* grad, void* param_lp, DType lp_dt, long long n, cudaStream_t s);
// dst(dt) = src(fp32)
cudaError_t cast_from_f32(DType dt, const float* src, void* dst, long long n, cudaStream_t s);

// dst[i] = sum over r < world (in rank order) of src.p[r][i]; the sources
// are peers' buffers mapped through CUDA IPC (kernels/peer.cu)
constexpr int kMaxPeers = 8;
struct PeerSrcs {
  const float* p[kMaxPeers];
};
cudaError_t peer_sum(const PeerSrcs& src, int world, float* dst, long long n, cudaStream_t s);
// cross-rank counters (engine/peer_comm.hpp): release-store `value` into n
// counters / spin (acquire) until n counters reach `value`
struct PeerFlags {
  uint32_t* p[kMaxPeers];
};
cudaError_t peer_signal(const PeerFlags& f, int n, uint32_t value, cudaStream_t s);
cudaError_t peer_wait_spin(const PeerFlags& f, int n, uint32_t value, cudaStream_t s);

}  // namespace gs
