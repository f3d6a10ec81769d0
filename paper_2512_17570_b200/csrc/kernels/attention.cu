// Causal multi-head attention of the layer executor (forward with saved
// log-sum-exp, recompute-based backward).
//
//  * bf16, head_dim in {64,128}, s % 64 == 0: flash-attention tiling on the
//    tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate, online softmax in
//    registers, ldmatrix operand loads from padded shared memory, cp.async
//    double-buffered K/V streaming).  Backward walks key blocks per CTA,
//    accumulates dK/dV in registers and dQ with fp32 red.add.
//  * otherwise (fp32 parity mode, tiny heads): warp-per-query SIMT kernels,
//    fp32 math throughout.
// qkv layout [b*s][3h]: q | k | v column blocks, head j at columns j*d.
#include "common.cuh"
#include "kernels.h"

namespace gs {

namespace {

using bf16 = __nv_bfloat16;

// =============================================================== SIMT path
template <typename T>
__global__ void __launch_bounds__(128) attn_fwd_simt(const T* __restrict__ qkv, T* __restrict__ o,
                                                     float* __restrict__ lse, int b, int s, int h, int H,
                                                     float scale) {
  __shared__ float qs[4][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * 4 + warp;
  if (gw >= (long long)b * H * s) return;
  const int d = h / H;
  const int bh = (int)(gw / s), t = (int)(gw % s);
  const int bi = bh / H, j = bh % H;
  const long long ld3 = 3LL * h;
  const T* qrow = qkv + ((long long)bi * s + t) * ld3 + j * d;
  for (int e = lane; e < d; e += 32) qs[warp][e] = ld(qrow + e);
  __syncwarp();
  float m = -INFINITY, l = 0.0f, acc[4] = {0, 0, 0, 0};
  for (int u0 = 0; u0 <= t; u0 += 32) {
    const int u = u0 + lane;
    float sc = -INFINITY;
    if (u <= t) {
      const T* krow = qkv + ((long long)bi * s + u) * ld3 + h + j * d;
      float a = 0.0f;
      for (int e = 0; e < d; ++e) a = fmaf(qs[warp][e], ld(krow + e), a);
      sc = a * scale;
    }
    const float mn = fmaxf(m, warp_max(sc));
    const float p = u <= t ? expf(sc - mn) : 0.0f;
    const float corr = expf(m - mn);
    l = l * corr + warp_sum(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] *= corr;
    const int cnt = min(32, t - u0 + 1);
    for (int kk = 0; kk < cnt; ++kk) {
      const float pk = __shfl_sync(0xffffffffu, p, kk);
      const T* vrow = qkv + ((long long)bi * s + u0 + kk) * ld3 + 2 * h + j * d;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = lane + 32 * k;
        if (e < d) acc[k] = fmaf(pk, ld(vrow + e), acc[k]);
      }
    }
    m = mn;
  }
  T* orow = o + ((long long)bi * s + t) * h + j * d;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = lane + 32 * k;
    if (e < d) st(orow + e, acc[k] / l);
  }
  if (lane == 0) lse[(long long)bh * s + t] = m + logf(l);
}

// dk/dv accumulate into fp32 workspace kv[b*s][2h]; dq written directly.
template <typename T>
__global__ void __launch_bounds__(128) attn_bwd_simt(const T* __restrict__ qkv, const T* __restrict__ o,
                                                     const float* __restrict__ lse, const T* __restrict__ dout,
                                                     T* __restrict__ dqkv, float* __restrict__ kv, int b, int s,
                                                     int h, int H, float scale) {
  __shared__ float qs[4][128], dos[4][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * 4 + warp;
  if (gw >= (long long)b * H * s) return;
  const int d = h / H;
  const int bh = (int)(gw / s), t = (int)(gw % s);
  const int bi = bh / H, j = bh % H;
  const long long ld3 = 3LL * h;
  const long long row_t = (long long)bi * s + t;
  float Dt = 0.0f;
  for (int e = lane; e < d; e += 32) {
    qs[warp][e] = ld(qkv + row_t * ld3 + j * d + e);
    const float g = ld(dout + row_t * h + j * d + e);
    dos[warp][e] = g;
    Dt += g * ld(o + row_t * h + j * d + e);
  }
  Dt = warp_sum(Dt);
  __syncwarp();
  const float L = lse[(long long)bh * s + t];
  float dq[4] = {0, 0, 0, 0};
  for (int u0 = 0; u0 <= t; u0 += 32) {
    const int u = u0 + lane;
    float p = 0.0f, ds = 0.0f;
    if (u <= t) {
      const T* krow = qkv + ((long long)bi * s + u) * ld3 + h + j * d;
      const T* vrow = krow + h;
      float sc = 0.0f, dp = 0.0f;
      for (int e = 0; e < d; ++e) {
        sc = fmaf(qs[warp][e], ld(krow + e), sc);
        dp = fmaf(dos[warp][e], ld(vrow + e), dp);
      }
      p = expf(sc * scale - L);
      ds = p * (dp - Dt);
    }
    const int cnt = min(32, t - u0 + 1);
    for (int kk = 0; kk < cnt; ++kk) {
      const float pk = __shfl_sync(0xffffffffu, p, kk);
      const float dk = __shfl_sync(0xffffffffu, ds, kk) * scale;
      const long long row_u = (long long)bi * s + u0 + kk;
      const T* krow = qkv + row_u * ld3 + h + j * d;
      float* kvrow = kv + row_u * 2 * h + j * d;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = lane + 32 * k;
        if (e < d) {
          dq[k] = fmaf(dk, ld(krow + e), dq[k]);
          atomicAdd(kvrow + e, dk * qs[warp][e]);
          atomicAdd(kvrow + h + e, pk * dos[warp][e]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = lane + 32 * k;
    if (e < d) st(dqkv + row_t * ld3 + j * d + e, dq[k]);
  }
}

template <typename T>
__global__ void kv_store_kernel(const float* __restrict__ kv, T* __restrict__ dqkv, long long rows, int h) {
  const long long n = rows * 2LL * h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / (2LL * h), c = i % (2LL * h);
    st(dqkv + r * 3LL * h + h + c, kv[i]);
  }
}

// ========================================================= tensor-core path
constexpr int kFaBM = 64;   // queries per forward CTA (4 warps x 16 rows)
constexpr int kFaBN = 64;   // keys per block
constexpr int kFaBQ = 32;   // queries per backward step
constexpr int kPad = 8;     // bf16 elements of row padding (bank-conflict-free ldmatrix)

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ldsm4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr(p)));
}
__device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// rows x HD tile from global rows (stride ld elements) into padded smem.
template <int HD, int ROWS>
__device__ __forceinline__ void load_tile(bf16* dst, const bf16* src, long long ld) {
  constexpr int kChunks = HD / 8;  // 16-byte chunks per row
  for (int c = threadIdx.x; c < ROWS * kChunks; c += blockDim.x) {
    const int r = c / kChunks, k = c % kChunks;
    cp_async16(dst + r * (HD + kPad) + k * 8, src + r * ld + k * 8);
  }
}

// A fragment (16 rows x 16 k) from row-major smem [row][k] (row stride lds).
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const bf16* base, int lds, int lane) {
  const int mi = lane >> 3;
  ldsm4(a, base + ((lane & 7) + 8 * (mi & 1)) * lds + 8 * (mi >> 1));
}
// Two n-tiles of B fragments from smem stored [n][k] (k contiguous).
__device__ __forceinline__ void frag_b_nk(uint32_t (&b)[4], const bf16* base, int lds, int lane) {
  const int mi = lane >> 3;
  ldsm4(b, base + ((lane & 7) + 8 * (mi >> 1)) * lds + 8 * (mi & 1));
}
// Two n-tiles of B fragments from smem stored [k][n] (n contiguous).
__device__ __forceinline__ void frag_b_kn(uint32_t (&b)[4], const bf16* base, int lds, int lane) {
  const int mi = lane >> 3;
  ldsm4t(b, base + ((lane & 7) + 8 * (mi & 1)) * lds + 8 * (mi >> 1));
}
// A fragment (16 m x 16 k) from smem stored [k][m] (m contiguous).
__device__ __forceinline__ void frag_a_km(uint32_t (&a)[4], const bf16* base, int lds, int lane) {
  const int mi = lane >> 3;
  ldsm4t(a, base + ((lane & 7) + 8 * (mi >> 1)) * lds + 8 * (mi & 1));
}

template <int HD>
__global__ void __launch_bounds__(128) fa_fwd_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ o,
                                                     float* __restrict__ lse, int s, int h, int H, float scale) {
  constexpr int LDS = HD + kPad;
  extern __shared__ __align__(16) uint8_t fa_smem[];
  bf16* Qs = reinterpret_cast<bf16*>(fa_smem);
  bf16* Ks = Qs + kFaBM * LDS;          // 2 buffers
  bf16* Vs = Ks + 2 * kFaBN * LDS;      // 2 buffers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int qb = gridDim.x - 1 - blockIdx.x;  // heavy (late) query blocks first
  const int bh = blockIdx.y, bi = bh / H, j = bh % H;
  const long long ld3 = 3LL * h;
  const bf16* base = qkv + (long long)bi * s * ld3 + j * HD;
  const int q0 = qb * kFaBM;

  load_tile<HD, kFaBM>(Qs, base + (long long)q0 * ld3, ld3);
  load_tile<HD, kFaBN>(Ks, base + h, ld3);
  load_tile<HD, kFaBN>(Vs, base + 2 * h, ld3);
  cp_async_commit();

  float oacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.0f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.0f, 0.0f};
  uint32_t qf[HD / 16][4];
  const float sl2 = scale * 1.4426950408889634f;  // scores in log2 units

  for (int kb = 0; kb <= qb; ++kb) {
    const int buf = kb & 1;
    if (kb < qb) {  // prefetch the next K/V block
      load_tile<HD, kFaBN>(Ks + (buf ^ 1) * kFaBN * LDS, base + (long long)(kb + 1) * kFaBN * ld3 + h, ld3);
      load_tile<HD, kFaBN>(Vs + (buf ^ 1) * kFaBN * LDS, base + (long long)(kb + 1) * kFaBN * ld3 + 2 * h, ld3);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) frag_a(qf[kk], Qs + (warp * 16) * LDS + kk * 16, LDS, lane);
    }
    const bf16* K = Ks + buf * kFaBN * LDS;
    const bf16* V = Vs + buf * kFaBN * LDS;
    float sc[kFaBN / 8][4];
#pragma unroll
    for (int i = 0; i < kFaBN / 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
      for (int p = 0; p < kFaBN / 16; ++p) {
        uint32_t bfr[4];
        frag_b_nk(bfr, K + (p * 16) * LDS + kk * 16, LDS, lane);
        mma16816(sc[2 * p], qf[kk], bfr[0], bfr[1]);
        mma16816(sc[2 * p + 1], qf[kk], bfr[2], bfr[3]);
      }
    // causal mask on the diagonal block, then online softmax (log2 domain)
    const int row0 = q0 + warp * 16 + g;
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int nt = 0; nt < kFaBN / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = kb * kFaBN + nt * 8 + 2 * tq + (e & 1);
        const int row = row0 + (e >> 1) * 8;
        float v = sc[nt][e] * sl2;
        if (kb == qb && col > row) v = -INFINITY;
        sc[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.0f, 0.0f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = exp2f(mrow[r] - mx[r]);
#pragma unroll
    for (int nt = 0; nt < kFaBN / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(sc[nt][e] - mx[e >> 1]);
        sc[nt][e] = p;
        rs[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lrow[r] = lrow[r] * corr[r] + rs[r];
      mrow[r] = mx[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      oacc[i][0] *= corr[0];
      oacc[i][1] *= corr[0];
      oacc[i][2] *= corr[1];
      oacc[i][3] *= corr[1];
    }
    // O += P V  (P from registers, V fragments via ldmatrix.trans)
#pragma unroll
    for (int kk = 0; kk < kFaBN / 16; ++kk) {
      uint32_t pa[4] = {pack2(sc[2 * kk][0], sc[2 * kk][1]), pack2(sc[2 * kk][2], sc[2 * kk][3]),
                        pack2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]), pack2(sc[2 * kk + 1][2], sc[2 * kk + 1][3])};
#pragma unroll
      for (int p = 0; p < HD / 16; ++p) {
        uint32_t bfr[4];
        frag_b_kn(bfr, V + (kk * 16) * LDS + p * 16, LDS, lane);
        mma16816(oacc[2 * p], pa, bfr[0], bfr[1]);
        mma16816(oacc[2 * p + 1], pa, bfr[2], bfr[3]);
      }
    }
    __syncthreads();  // buffer reuse by the next prefetch
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const int row_a = q0 + warp * 16 + g;
  bf16* obase = o + ((long long)bi * s) * h + j * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(obase + (long long)row_a * h + col) = pack2(oacc[i][0] / lrow[0], oacc[i][1] / lrow[0]);
    *reinterpret_cast<uint32_t*>(obase + (long long)(row_a + 8) * h + col) =
        pack2(oacc[i][2] / lrow[1], oacc[i][3] / lrow[1]);
  }
  if (tq == 0) {
    const float ln2 = 0.6931471805599453f;
    lse[(long long)bh * s + row_a] = (mrow[0] + log2f(lrow[0])) * ln2;
    lse[(long long)bh * s + row_a + 8] = (mrow[1] + log2f(lrow[1])) * ln2;
  }
}

// D[bh][q] = sum_e dO[q, head] * O[q, head]
template <int HD>
__global__ void fa_dot_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ D,
                              int b, int s, int h, int H) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + warp;
  if (gw >= (long long)b * H * s) return;
  const int bh = (int)(gw / s), t = (int)(gw % s), bi = bh / H, j = bh % H;
  const long long off = ((long long)bi * s + t) * h + j * HD;
  float acc = 0.0f;
  for (int e = lane; e < HD; e += 32) acc += __bfloat162float(o[off + e]) * __bfloat162float(dout[off + e]);
  acc = warp_sum(acc);
  if (lane == 0) D[gw] = acc;
}

template <int HD>
__global__ void __launch_bounds__(128, 1) fa_bwd_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                        const float* __restrict__ lse, const float* __restrict__ Dg,
                                                        bf16* __restrict__ dqkv, float* __restrict__ dq_acc, int s,
                                                        int h, int H, float scale) {
  constexpr int LDS = HD + kPad;
  constexpr int LDP = kFaBQ + kPad;
  extern __shared__ __align__(16) uint8_t fa_smem[];
  bf16* Ks = reinterpret_cast<bf16*>(fa_smem);
  bf16* Vs = Ks + kFaBN * LDS;
  bf16* Qs = Vs + kFaBN * LDS;            // 2 buffers of kFaBQ rows
  bf16* dOs = Qs + 2 * kFaBQ * LDS;       // 2 buffers
  bf16* dSs = dOs + 2 * kFaBQ * LDS;      // [key 64][query kFaBQ] (dS^T)
  float* Ls = reinterpret_cast<float*>(dSs + kFaBN * LDP);  // 2 x kFaBQ
  float* Ds = Ls + 2 * kFaBQ;                               // 2 x kFaBQ

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, bi = bh / H, j = bh % H;
  const long long ld3 = 3LL * h;
  const bf16* qbase = qkv + (long long)bi * s * ld3 + j * HD;
  const bf16* dobase = dout + (long long)bi * s * h + j * HD;
  const int k0 = kb * kFaBN;
  const float sl2 = scale * 1.4426950408889634f;
  const float log2e = 1.4426950408889634f;

  load_tile<HD, kFaBN>(Ks, qbase + (long long)k0 * ld3 + h, ld3);
  load_tile<HD, kFaBN>(Vs, qbase + (long long)k0 * ld3 + 2 * h, ld3);
  const int nq = (s - k0) / kFaBQ;  // query blocks from the diagonal down
  auto issue_q = [&](int i, int buf) {
    const int q0 = k0 + i * kFaBQ;
    load_tile<HD, kFaBQ>(Qs + buf * kFaBQ * LDS, qbase + (long long)q0 * ld3, ld3);
    load_tile<HD, kFaBQ>(dOs + buf * kFaBQ * LDS, dobase + (long long)q0 * h, h);
    for (int r = threadIdx.x; r < kFaBQ; r += blockDim.x) {
      Ls[buf * kFaBQ + r] = lse[(long long)bh * s + q0 + r] * log2e;
      Ds[buf * kFaBQ + r] = Dg[(long long)bh * s + q0 + r];
    }
  };
  issue_q(0, 0);
  cp_async_commit();

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.0f;

  const bf16* Kw = Ks + (warp * 16) * LDS;  // this warp's 16 keys
  const bf16* Vw = Vs + (warp * 16) * LDS;
  for (int i = 0; i < nq; ++i) {
    const int buf = i & 1;
    if (i + 1 < nq) {
      issue_q(i + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const bf16* Q = Qs + buf * kFaBQ * LDS;
    const bf16* dO = dOs + buf * kFaBQ * LDS;
    const float* L = Ls + buf * kFaBQ;
    const float* Dq = Ds + buf * kFaBQ;
    const int q0 = k0 + i * kFaBQ;
    // S^T = K Q^T and dP^T = V dO^T : [16 keys x kFaBQ queries] per warp
    float st[kFaBQ / 8][4], dpt[kFaBQ / 8][4];
#pragma unroll
    for (int n = 0; n < kFaBQ / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[n][e] = dpt[n][e] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ka[4], va[4];
      frag_a(ka, Kw + kk * 16, LDS, lane);
      frag_a(va, Vw + kk * 16, LDS, lane);
#pragma unroll
      for (int p = 0; p < kFaBQ / 16; ++p) {
        uint32_t qb_[4], db_[4];
        frag_b_nk(qb_, Q + (p * 16) * LDS + kk * 16, LDS, lane);
        frag_b_nk(db_, dO + (p * 16) * LDS + kk * 16, LDS, lane);
        mma16816(st[2 * p], ka, qb_[0], qb_[1]);
        mma16816(st[2 * p + 1], ka, qb_[2], qb_[3]);
        mma16816(dpt[2 * p], va, db_[0], db_[1]);
        mma16816(dpt[2 * p + 1], va, db_[2], db_[3]);
      }
    }
    // P^T, dS^T (rows = keys, cols = queries)
    const int key_a = k0 + warp * 16 + g;
#pragma unroll
    for (int n = 0; n < kFaBQ / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = n * 8 + 2 * tq + (e & 1);
        const int key = key_a + (e >> 1) * 8;
        float p = exp2f(st[n][e] * sl2 - L[qc]);
        if (q0 + qc < key) p = 0.0f;
        st[n][e] = p;
        dpt[n][e] = p * (dpt[n][e] - Dq[qc]);
      }
    // dV += P^T dO ; dK += dS^T Q   (A from registers, B = [query][d] via trans)
#pragma unroll
    for (int kk = 0; kk < kFaBQ / 16; ++kk) {
      const uint32_t pa[4] = {pack2(st[2 * kk][0], st[2 * kk][1]), pack2(st[2 * kk][2], st[2 * kk][3]),
                              pack2(st[2 * kk + 1][0], st[2 * kk + 1][1]), pack2(st[2 * kk + 1][2], st[2 * kk + 1][3])};
      const uint32_t sa[4] = {pack2(dpt[2 * kk][0], dpt[2 * kk][1]), pack2(dpt[2 * kk][2], dpt[2 * kk][3]),
                              pack2(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]),
                              pack2(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3])};
#pragma unroll
      for (int p = 0; p < HD / 16; ++p) {
        uint32_t bo[4], bq[4];
        frag_b_kn(bo, dO + (kk * 16) * LDS + p * 16, LDS, lane);
        frag_b_kn(bq, Q + (kk * 16) * LDS + p * 16, LDS, lane);
        mma16816(dv[2 * p], pa, bo[0], bo[1]);
        mma16816(dv[2 * p + 1], pa, bo[2], bo[3]);
        mma16816(dk[2 * p], sa, bq[0], bq[1]);
        mma16816(dk[2 * p + 1], sa, bq[2], bq[3]);
      }
    }
    // stage dS^T for the dQ product
#pragma unroll
    for (int n = 0; n < kFaBQ / 8; ++n) {
      const int qc = n * 8 + 2 * tq;
      *reinterpret_cast<uint32_t*>(dSs + (warp * 16 + g) * LDP + qc) = pack2(dpt[n][0], dpt[n][1]);
      *reinterpret_cast<uint32_t*>(dSs + (warp * 16 + g + 8) * LDP + qc) = pack2(dpt[n][2], dpt[n][3]);
    }
    __syncthreads();
    // dQ[kFaBQ x HD] += dS K: warp w -> query m-tile (w & 1), d half (w >> 1)
    {
      const int mt = warp & 1, dh = warp >> 1;
      float dqa[HD / 16][4];
#pragma unroll
      for (int n = 0; n < HD / 16; ++n) dqa[n][0] = dqa[n][1] = dqa[n][2] = dqa[n][3] = 0.0f;
#pragma unroll
      for (int kk = 0; kk < kFaBN / 16; ++kk) {
        uint32_t a[4];
        frag_a_km(a, dSs + (kk * 16) * LDP + mt * 16, LDP, lane);
#pragma unroll
        for (int p = 0; p < HD / 32; ++p) {
          uint32_t bk[4];
          frag_b_kn(bk, Ks + (kk * 16) * LDS + dh * (HD / 2) + p * 16, LDS, lane);
          mma16816(dqa[2 * p], a, bk[0], bk[1]);
          mma16816(dqa[2 * p + 1], a, bk[2], bk[3]);
        }
      }
      const int qr = q0 + mt * 16 + g;
      float* dqb = dq_acc + ((long long)bi * s) * h + j * HD + dh * (HD / 2);
#pragma unroll
      for (int n = 0; n < HD / 16; ++n) {
        const int col = n * 8 + 2 * tq;
        atomicAdd(dqb + (long long)qr * h + col, dqa[n][0] * scale);
        atomicAdd(dqb + (long long)qr * h + col + 1, dqa[n][1] * scale);
        atomicAdd(dqb + (long long)(qr + 8) * h + col, dqa[n][2] * scale);
        atomicAdd(dqb + (long long)(qr + 8) * h + col + 1, dqa[n][3] * scale);
      }
    }
    __syncthreads();
  }
  // write dK (scaled), dV for this warp's 16 keys
  bf16* kout = dqkv + ((long long)bi * s) * ld3 + h + j * HD;
  const int kr = k0 + warp * 16 + g;
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    const int col = n * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(kout + (long long)kr * ld3 + col) = pack2(dk[n][0] * scale, dk[n][1] * scale);
    *reinterpret_cast<uint32_t*>(kout + (long long)(kr + 8) * ld3 + col) = pack2(dk[n][2] * scale, dk[n][3] * scale);
    *reinterpret_cast<uint32_t*>(kout + h + (long long)kr * ld3 + col) = pack2(dv[n][0], dv[n][1]);
    *reinterpret_cast<uint32_t*>(kout + h + (long long)(kr + 8) * ld3 + col) = pack2(dv[n][2], dv[n][3]);
  }
}

__global__ void dq_store_kernel(const float* __restrict__ dq, bf16* __restrict__ dqkv, long long rows, int h) {
  const long long n = rows * h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / h, c = i % h;
    dqkv[r * 3LL * h + c] = __float2bfloat16_rn(dq[i]);
  }
}

// Vectorised backward prologue / epilogue of the tcgen05 path (h % 8 == 0,
// head_dim 128): D = rowsum(dO * O) per (bh, query) with 16 lanes per row
// (8 bf16 each, 16-byte loads) and L2 = lse * log2(e); the same pass zeroes
// the fp32 dQ accumulator the kernel reduce-adds into (no separate memset).
__global__ void fa_prep_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, const float* __restrict__ lse,
                               float* __restrict__ D, float* __restrict__ L2, float* __restrict__ dq, int b, int s,
                               int h, int H) {
  pdl_trigger_and_wait();
  const long long rows = (long long)b * H * s;
  const int sub = threadIdx.x & 15;
  for (long long gr = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4; gr < rows;
       gr += ((long long)gridDim.x * blockDim.x) >> 4) {
    const int bh = (int)(gr / s), t = (int)(gr % s), bi = bh / H, j = bh % H;
    const long long off = ((long long)bi * s + t) * h + j * 128 + sub * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(o + off);
    const uint4 g = *reinterpret_cast<const uint4*>(dout + off);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pg = reinterpret_cast<const __nv_bfloat162*>(&g);
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fa = __bfloat1622float2(pa[k]), fg = __bfloat1622float2(pg[k]);
      acc += fa.x * fg.x + fa.y * fg.y;
    }
#pragma unroll
    for (int m = 8; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (sub == 0) {
      D[gr] = acc;
      L2[gr] = lse[gr] * 1.4426950408889634f;  // log2-domain lse for the SFU exp2
    }
    float4* z = reinterpret_cast<float4*>(dq + off);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dQ fp32 [b*s][h] -> bf16 q-columns of dqkv [b*s][3h], 8 columns per thread.
__global__ void dq_store_vec_kernel(const float* __restrict__ dq, bf16* __restrict__ dqkv, long long rows, int h) {
  pdl_trigger_and_wait();
  const long long n8 = rows * h / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 8, r = e / h, c = e % h;
    const float4 x = *reinterpret_cast<const float4*>(dq + e);
    const float4 y = *reinterpret_cast<const float4*>(dq + e + 4);
    __nv_bfloat162 v[4] = {__floats2bfloat162_rn(x.x, x.y), __floats2bfloat162_rn(x.z, x.w),
                           __floats2bfloat162_rn(y.x, y.y), __floats2bfloat162_rn(y.z, y.w)};
    *reinterpret_cast<uint4*>(dqkv + r * 3LL * h + c) = *reinterpret_cast<const uint4*>(v);
  }
}

bool fa_ok(DType dt, int s, int h, int H) {
  if (dt != DType::BF16) return false;
  const int d = h / H;
  return (d == 64 || d == 128) && s % kFaBM == 0 && h % 8 == 0;
}
template <int HD> constexpr int fwd_smem() { return (kFaBM + 4 * kFaBN) * (HD + kPad) * 2; }
template <int HD> constexpr int bwd_smem() {
  return (2 * kFaBN + 4 * kFaBQ) * (HD + kPad) * 2 + kFaBN * (kFaBQ + kPad) * 2 + 4 * kFaBQ * 4;
}

template <int HD>
cudaError_t fa_fwd(const bf16* qkv, bf16* o, float* lse, int b, int s, int h, int H, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(fa_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem<HD>());
    if (e != cudaSuccess) return e;
    init = true;
  }
  const dim3 grid(s / kFaBM, b * H);
  count_launch(); fa_fwd_kernel<HD><<<grid, 128, fwd_smem<HD>(), st>>>(qkv, o, lse, s, h, H, 1.0f / sqrtf((float)HD));
  return cudaGetLastError();
}

template <int HD>
cudaError_t fa_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv, void* work,
                   int b, int s, int h, int H, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(fa_bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, bwd_smem<HD>());
    if (e != cudaSuccess) return e;
    init = true;
  }
  float* dq = static_cast<float*>(work);
  float* D = dq + (size_t)b * s * h;
  float* L2 = D + (size_t)b * H * s;
  const long long rows = (long long)b * H * s;
  cudaError_t e = cudaSuccess;
  if (HD == 128 && attention_tc_supported(DType::BF16, s, h, H)) {
    count_launch();
    e = launch_pdl(fa_prep_kernel, dim3(grid_for(rows * 16, 256)), dim3(256), 0, st, (const bf16*)o,
                   (const bf16*)dout, lse, D, L2, dq, b, s, h, H);
    if (e != cudaSuccess) return e;
    e = attention_bwd_tc(qkv, dout, lse, L2, D, dqkv, dq, b, s, h, H, st);
    if (e != cudaSuccess) return e;
    count_launch();
    return launch_pdl(dq_store_vec_kernel, dim3(grid_for((long long)b * s * h / 8, 256)), dim3(256), 0, st,
                      (const float*)dq, (bf16*)dqkv, (long long)b * s, h);
  }
  e = cudaMemsetAsync(dq, 0, sizeof(float) * (size_t)b * s * h, st);
  if (e != cudaSuccess) return e;
  count_launch(); fa_dot_kernel<HD><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(o, dout, D, b, s, h, H);
  {
    const dim3 grid(s / kFaBN, b * H);
    count_launch();
    fa_bwd_kernel<HD><<<grid, 128, bwd_smem<HD>(), st>>>(qkv, dout, lse, D, dqkv, dq, s, h, H, 1.0f / sqrtf((float)HD));
  }
  count_launch(); dq_store_kernel<<<grid_for((long long)b * s * h, 256, 4), 256, 0, st>>>(dq, dqkv, (long long)b * s, h);
  return cudaGetLastError();
}

}  // namespace

size_t attention_bwd_workspace(int b, int s, int h, int H) {
  // fa path: dq fp32 [b*s][h] + D, L2 [b*H*s];  simt path: dk|dv fp32 [b*s][2h]
  const size_t fa = sizeof(float) * ((size_t)b * s * h + 2 * (size_t)b * H * s);
  const size_t simt = sizeof(float) * (size_t)b * s * 2 * h;
  return fa > simt ? fa : simt;
}

cudaError_t attention_fwd(DType dt, const void* qkv, void* o, float* lse, int b, int s, int h, int H,
                          cudaStream_t st) {
  if (h % H || h / H > 128) return cudaErrorInvalidValue;
  if (attention_tc_supported(dt, s, h, H)) return attention_fwd_tc(qkv, o, lse, b, s, h, H, st);
  if (fa_ok(dt, s, h, H)) {
    if (h / H == 128) return fa_fwd<128>((const bf16*)qkv, (bf16*)o, lse, b, s, h, H, st);
    return fa_fwd<64>((const bf16*)qkv, (bf16*)o, lse, b, s, h, H, st);
  }
  const long long warps = (long long)b * H * s;
  const unsigned grid = (unsigned)((warps + 3) / 4);
  const float scale = 1.0f / sqrtf((float)(h / H));
  count_launch();
  if (dt == DType::F32)
    attn_fwd_simt<float><<<grid, 128, 0, st>>>((const float*)qkv, (float*)o, lse, b, s, h, H, scale);
  else
    attn_fwd_simt<bf16><<<grid, 128, 0, st>>>((const bf16*)qkv, (bf16*)o, lse, b, s, h, H, scale);
  return cudaGetLastError();
}

cudaError_t attention_bwd(DType dt, const void* qkv, const void* o, const float* lse, const void* dout, void* dqkv,
                          void* work, int b, int s, int h, int H, cudaStream_t st) {
  if (h % H || h / H > 128) return cudaErrorInvalidValue;
  if (fa_ok(dt, s, h, H)) {
    if (h / H == 128)
      return fa_bwd<128>((const bf16*)qkv, (const bf16*)o, lse, (const bf16*)dout, (bf16*)dqkv, work, b, s, h, H, st);
    return fa_bwd<64>((const bf16*)qkv, (const bf16*)o, lse, (const bf16*)dout, (bf16*)dqkv, work, b, s, h, H, st);
  }
  float* kv = static_cast<float*>(work);
  cudaError_t e = cudaMemsetAsync(kv, 0, sizeof(float) * (size_t)b * s * 2 * h, st);
  if (e != cudaSuccess) return e;
  const long long warps = (long long)b * H * s;
  const unsigned grid = (unsigned)((warps + 3) / 4);
  const float scale = 1.0f / sqrtf((float)(h / H));
  if (dt == DType::F32) {
    count_launch(); attn_bwd_simt<float><<<grid, 128, 0, st>>>((const float*)qkv, (const float*)o, lse, (const float*)dout,
                                               (float*)dqkv, kv, b, s, h, H, scale);
    count_launch(); kv_store_kernel<float><<<grid_for((long long)b * s * 2 * h, 256, 4), 256, 0, st>>>(kv, (float*)dqkv,
                                                                                        (long long)b * s, h);
  } else {
    count_launch(); attn_bwd_simt<bf16><<<grid, 128, 0, st>>>((const bf16*)qkv, (const bf16*)o, lse, (const bf16*)dout,
                                              (bf16*)dqkv, kv, b, s, h, H, scale);
    count_launch(); kv_store_kernel<bf16><<<grid_for((long long)b * s * 2 * h, 256, 4), 256, 0, st>>>(kv, (bf16*)dqkv,
                                                                                       (long long)b * s, h);
  }
  return cudaGetLastError();
}

}  // namespace gs
