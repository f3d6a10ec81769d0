// Causal multi-head attention of the layer executor (forward with saved
// log-sum-exp, recompute-based backward).
//
//  * bf16, head_dim 128, s % 256 == 0 (every BASELINE geometry): the tcgen05
//    flash-attention kernels of attention_tc.cu; this file holds their
//    vectorised backward prologue (D = rowsum(dO * O), log2-domain lse, dQ
//    accumulator zeroing) and epilogue (dQ fp32 -> bf16).
//  * otherwise (the fp32 parity mode, toy geometries): warp-per-query SIMT
//    kernels, fp32 math throughout.
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

// ============================================ tcgen05 path: prologue / epilogue
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

}  // namespace

size_t attention_bwd_workspace(int b, int s, int h, int H) {
  // tcgen05 path: dq fp32 [b*s][h] + D, L2 [b*H*s];  simt path: dk|dv fp32 [b*s][2h]
  const size_t fa = sizeof(float) * ((size_t)b * s * h + 2 * (size_t)b * H * s);
  const size_t simt = sizeof(float) * (size_t)b * s * 2 * h;
  return fa > simt ? fa : simt;
}

cudaError_t attention_fwd(DType dt, const void* qkv, void* o, float* lse, int b, int s, int h, int H,
                          cudaStream_t st) {
  if (h % H || h / H > 128) return cudaErrorInvalidValue;
  if (attention_tc_supported(dt, s, h, H)) return attention_fwd_tc(qkv, o, lse, b, s, h, H, st);
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
  if (attention_tc_supported(dt, s, h, H)) {
    // prologue (D, log2 lse, dQ zeroing) -> tcgen05 backward -> dQ to bf16
    float* dq = static_cast<float*>(work);
    float* D = dq + (size_t)b * s * h;
    float* L2 = D + (size_t)b * H * s;
    const long long rows = (long long)b * H * s;
    count_launch();
    cudaError_t e = launch_pdl(fa_prep_kernel, dim3(grid_for(rows * 16, 256)), dim3(256), 0, st, (const bf16*)o,
                               (const bf16*)dout, lse, D, L2, dq, b, s, h, H);
    if (e != cudaSuccess) return e;
    e = attention_bwd_tc(qkv, dout, lse, L2, D, dqkv, dq, b, s, h, H, st);
    if (e != cudaSuccess) return e;
    count_launch();
    return launch_pdl(dq_store_vec_kernel, dim3(grid_for((long long)b * s * h / 8, 256)), dim3(256), 0, st,
                      (const float*)dq, (bf16*)dqkv, (long long)b * s, h);
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
