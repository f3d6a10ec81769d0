// Row-wise and elementwise kernels of the layer executor: LayerNorm,
// GELU, residual add, embedding, softmax-cross-entropy and the fused chunked
// Adam step.  All HBM-bound: coalesced accesses, fp32 math, warp-shuffle +
// shared-memory block reductions, grids sized to the SM count.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cmath>

namespace gs {

namespace {

constexpr float kLnEps = 1e-5f;

// Block-wide sum for blockDim.x == 256 (8 warps); all threads get the result.
__device__ __forceinline__ float block_sum256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = l < 8 ? red[l] : 0.0f;
  return warp_sum(r);
}
__device__ __forceinline__ float block_max256(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = l < 8 ? red[l] : -INFINITY;
  return warp_max(r);
}

constexpr int kRowThreads = 256;
constexpr int kMaxPerThread = 48;  // h <= 12288

// Row kernels hold E = ceil(h / 256) values per thread in registers (E is a
// template parameter so occupancy follows h; a fixed 48-wide array for
// h <= 12288 left one block per SM and made these launches latency-bound).
template <typename T, int E>
__global__ void __launch_bounds__(kRowThreads) ln_fwd_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                             float* __restrict__ mean,
                                                             float* __restrict__ rstd, int h) {
  __shared__ float red[8];
  const long long row = blockIdx.x;
  const T* xr = x + row * h;
  float v[E];
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    v[k] = i < h ? ld(xr + i) : 0.0f;
    s += v[k];
  }
  const float mu = block_sum256(s, red) / h;
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < h) ss += (v[k] - mu) * (v[k] - mu);
  }
  const float rs = rsqrtf(block_sum256(ss, red) / h + kLnEps);
  T* yr = y + row * h;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < h) st(yr + i, (v[k] - mu) * rs);
  }
  if (threadIdx.x == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = rs;
  }
}

template <typename T, int E>
__global__ void __launch_bounds__(kRowThreads) ln_bwd_kernel(const T* __restrict__ x,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ rstd,
                                                             const T* __restrict__ dy, T* dx, int h,
                                                             bool accumulate) {
  __shared__ float red[8];
  const long long row = blockIdx.x;
  const float mu = mean[row], rs = rstd[row];
  const T* xr = x + row * h;
  const T* gr = dy + row * h;
  float xh[E], g[E];
  float sg = 0.0f, sgx = 0.0f;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    xh[k] = i < h ? (ld(xr + i) - mu) * rs : 0.0f;
    g[k] = i < h ? ld(gr + i) : 0.0f;
    sg += g[k];
    sgx += g[k] * xh[k];
  }
  const float mg = block_sum256(sg, red) / h;
  const float mgx = block_sum256(sgx, red) / h;
  T* dr = dx + row * h;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < h) {
      const float d = rs * (g[k] - mg - xh[k] * mgx);
      st(dr + i, accumulate ? ld(dr + i) + d : d);
    }
  }
}

// Vectorised row kernels (h % (16 / sizeof(T)) == 0, the engine's case): a
// row is owned by a group of nw warps sized so each lane holds at most C
// 16-byte vectors of every row operand — 4 in the forward (nw = 2 at h = 2048
// bf16, 8 at 8192), 2 in the backward (nw = 4 at 2048, 16 at 8192) — and
// blocks carry max(1, 8 / nw) rows.  Small C keeps the register footprint at
// ~40-60 (the earlier one-warp-per-row shape held 8 vectors per operand,
// 137-174 registers, one CTA per SM, and ran latency-bound at 0.33-0.50 of
// HBM; its h > 4096 instance spilled).
template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void unpack(const uint4& r, float* f) {
    f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
  }
  __device__ __forceinline__ static uint4 pack(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
  __device__ __forceinline__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
  __device__ __forceinline__ static void unpack(const uint4& r, float* f) {
    f[0] = lo(r.x); f[1] = hi(r.x); f[2] = lo(r.y); f[3] = hi(r.y);
    f[4] = lo(r.z); f[5] = hi(r.z); f[6] = lo(r.w); f[7] = hi(r.w);
  }
  __device__ __forceinline__ static uint32_t p2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __device__ __forceinline__ static uint4 pack(const float* f) {
    return make_uint4(p2(f[0], f[1]), p2(f[2], f[3]), p2(f[4], f[5]), p2(f[6], f[7]));
  }
};

// Sum over the nw warps of this thread's row group (uniform nw per launch);
// float2 so the backward's two row sums share one pass of barriers.
__device__ __forceinline__ float2 group_sum2(float2 v, float2* red, int nw) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  if (nw == 1) return v;
  const int w = threadIdx.x >> 5, base = (w / nw) * nw;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float2 r = make_float2(0.0f, 0.0f);
  for (int i = 0; i < nw; ++i) {
    const float2 q = red[base + i];
    r.x += q.x;
    r.y += q.y;
  }
  return r;
}

constexpr int kVecRowMaxThreads = 512;

// One reduction per row: sums of (x - K) and (x - K)^2 with the shift K =
// x[row][0] (broadcast from lane 0's first vector), so the variance is
// E[(x-K)^2] - E[x-K]^2 without the cancellation of the unshifted one-pass
// form, and the row needs a single float2 group sum (one barrier pair when
// nw > 1) instead of the two-pass form's two.
template <typename T, int C>
__global__ void __launch_bounds__(kVecRowMaxThreads) ln_fwd_vec_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                                       float* __restrict__ mean,
                                                                       float* __restrict__ rstd, int rows, int h,
                                                                       int nw) {
  pdl_trigger_and_wait();
  using VT = Vec<T>;
  constexpr int N = VT::N;
  __shared__ float2 red[kVecRowMaxThreads / 32];
  const int gt = 32 * nw, t = threadIdx.x % gt;
  const long long row = (long long)blockIdx.x * (blockDim.x / gt) + threadIdx.x / gt;
  const bool live = row < rows;
  const int nv = h / N;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
  uint4 raw[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const int v = t + k * gt;
    raw[k] = (live && v < nv) ? __ldg(xr + v) : make_uint4(0, 0, 0, 0);
  }
  const float K = live ? ld(x + row * h) : 0.0f;  // the row's first element (an L1 hit)
  float s = 0.0f, ss = 0.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    if (t + k * gt < nv) {
      float f[N];
      VT::unpack(raw[k], f);
#pragma unroll
      for (int e = 0; e < N; ++e) {
        const float d = f[e] - K;
        s += d;
        ss += d * d;
      }
    }
  }
  const float2 m = group_sum2(make_float2(s, ss), red, nw);
  const float md = m.x / h;
  const float mu = K + md;
  const float rs = rsqrtf(fmaxf(m.y / h - md * md, 0.0f) + kLnEps);
  if (!live) return;
  uint4* yr = reinterpret_cast<uint4*>(y + row * h);
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const int v = t + k * gt;
    if (v < nv) {
      float f[N];
      VT::unpack(raw[k], f);
#pragma unroll
      for (int e = 0; e < N; ++e) f[e] = (f[e] - mu) * rs;
      yr[v] = VT::pack(f);
    }
  }
  if (t == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = rs;
  }
}

// dx = res + rs * (g - mean(g) - xh * mean(g * xh)); res may alias dx or be null.
// The residual's loads are issued with x and dy, ahead of the row reduction.
template <typename T, int C>
__global__ void __launch_bounds__(kVecRowMaxThreads) ln_bwd_vec_kernel(const T* __restrict__ x,
                                                                       const float* __restrict__ mean,
                                                                       const float* __restrict__ rstd,
                                                                       const T* __restrict__ dy, const T* res, T* dx,
                                                                       int rows, int h, int nw) {
  pdl_trigger_and_wait();
  using VT = Vec<T>;
  constexpr int N = VT::N;
  __shared__ float2 red[kVecRowMaxThreads / 32];
  const int gt = 32 * nw, t = threadIdx.x % gt;
  const long long row = (long long)blockIdx.x * (blockDim.x / gt) + threadIdx.x / gt;
  const bool live = row < rows;
  const int nv = h / N;
  const float mu = live ? mean[row] : 0.0f, rs = live ? rstd[row] : 0.0f;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
  const uint4* gr = reinterpret_cast<const uint4*>(dy + row * h);
  const uint4* rr = reinterpret_cast<const uint4*>(res + row * h);
  uint4 rx[C], rg[C], rres[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const int v = t + k * gt;
    const bool ok = live && v < nv;
    rx[k] = ok ? __ldg(xr + v) : make_uint4(0, 0, 0, 0);
    rg[k] = ok ? __ldg(gr + v) : make_uint4(0, 0, 0, 0);
    rres[k] = (ok && res) ? rr[v] : make_uint4(0, 0, 0, 0);
  }
  float sg = 0.0f, sgx = 0.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    float fx[N], fg[N];
    VT::unpack(rx[k], fx);
    VT::unpack(rg[k], fg);
#pragma unroll
    for (int e = 0; e < N; ++e) {
      sg += fg[e];
      sgx += fg[e] * ((fx[e] - mu) * rs);
    }
  }
  const float2 m = group_sum2(make_float2(sg, sgx), red, nw);
  const float mg = m.x / h, mgx = m.y / h;
  if (!live) return;
  uint4* dr = reinterpret_cast<uint4*>(dx + row * h);
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const int v = t + k * gt;
    if (v < nv) {
      float fx[N], fg[N], fr[N];
      VT::unpack(rx[k], fx);
      VT::unpack(rg[k], fg);
      VT::unpack(rres[k], fr);
#pragma unroll
      for (int e = 0; e < N; ++e) fx[e] = fr[e] + rs * (fg[e] - mg - ((fx[e] - mu) * rs) * mgx);
      dr[v] = VT::pack(fx);
    }
  }
}

struct RowShape {
  int nw, rpb, c;  // warps per row (<= 16), rows per block, 16-byte vectors per lane (<= 8 for h <= 12288)
};
// per_lane: target 16-byte vectors per lane and row operand (forward 4: one
// row operand, a single reduction; backward 2: x, dy and the residual live
// across the reduction)
inline RowShape row_shape(int h, int n, int per_lane) {
  const int nv = h / n;
  RowShape r;
  r.nw = std::min(kVecRowMaxThreads / 32, std::max(1, (nv + 32 * per_lane - 1) / (32 * per_lane)));
  r.rpb = std::max(1, 8 / r.nw);
  r.c = (nv + 32 * r.nw - 1) / (32 * r.nw);
  return r;
}
#define GS_TRY_E(expr)                      \
  do {                                      \
    const cudaError_t e_ = (expr);          \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)

#define GS_ROW_C(c, ...)                                       \
  do {                                                         \
    if ((c) <= 1) { constexpr int C = 1; __VA_ARGS__; }        \
    else if ((c) <= 2) { constexpr int C = 2; __VA_ARGS__; }   \
    else if ((c) <= 4) { constexpr int C = 4; __VA_ARGS__; }   \
    else { constexpr int C = 32 / Vec<T>::N; __VA_ARGS__; }    \
  } while (0)

// E in {1,2,4,8,16,24,32,48}: smallest covering h
#define GS_ROW_E(h, ...)                                  \
  do {                                                    \
    const int e_ = ((h) + kRowThreads - 1) / kRowThreads; \
    if (e_ <= 1) { constexpr int E = 1; __VA_ARGS__; }    \
    else if (e_ <= 2) { constexpr int E = 2; __VA_ARGS__; } \
    else if (e_ <= 4) { constexpr int E = 4; __VA_ARGS__; } \
    else if (e_ <= 8) { constexpr int E = 8; __VA_ARGS__; } \
    else if (e_ <= 16) { constexpr int E = 16; __VA_ARGS__; } \
    else if (e_ <= 24) { constexpr int E = 24; __VA_ARGS__; } \
    else if (e_ <= 32) { constexpr int E = 32; __VA_ARGS__; } \
    else { constexpr int E = 48; __VA_ARGS__; }           \
  } while (0)

template <typename T>
__global__ void gelu_fwd_kernel(const T* __restrict__ u, T* __restrict__ g, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    st(g + i, gelu_f(ld(u + i)));
}
template <typename T>
__global__ void gelu_bwd_kernel(const T* __restrict__ u, const T* dg, T* du, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    st(du + i, ld(dg + i) * gelu_grad_f(ld(u + i)));
}
template <typename T>
__global__ void add_kernel(const T* a, const T* b, T* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    st(y + i, ld(a + i) + ld(b + i));
}

template <typename T>
__global__ void embed_fwd_kernel(const T* __restrict__ wte, const T* __restrict__ wpe,
                                 const int32_t* __restrict__ tok, T* __restrict__ x0, int s, int h) {
  const int row = blockIdx.x;  // bi*s + t
  const int bi = row / s, t = row % s;
  const long long id = tok[bi * (s + 1) + t];
  for (int i = threadIdx.x; i < h; i += blockDim.x)
    st(x0 + (long long)row * h + i, ld(wte + id * h + i) + ld(wpe + (long long)t * h + i));
}
template <typename T>
__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const T* __restrict__ dx0,
                                 float* dwte, float* dwpe, int s, int h) {
  const int row = blockIdx.x;
  const int bi = row / s, t = row % s;
  const long long id = tok[bi * (s + 1) + t];
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const float g = ld(dx0 + (long long)row * h + i);
    atomicAdd(dwte + id * h + i, g);
    atomicAdd(dwpe + (long long)t * h + i, g);
  }
}

template <typename T>
__device__ __forceinline__ void st4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void st4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
  __nv_bfloat162 v[2] = {__floats2bfloat162_rn(a, b), __floats2bfloat162_rn(c, d)};
  *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(v);
}

// One row (token) per block.  Pass 1: each thread keeps an online (max, sum
// of exp) over its 16-byte vectors, combined across the block; pass 2 writes
// d(CE)/dlogits = (softmax - onehot) * scale.  The row is read twice (the
// second read mostly from L2) instead of three times; SFU exponentials
// (__expf, relative error ~2^-21), libm log for the loss.
__device__ __forceinline__ void online_add(float& m, float& z, float x) {
  if (x > m) {
    z = z * __expf(m - x) + 1.0f;
    m = x;
  } else {
    z += __expf(x - m);
  }
}
template <typename T>
__global__ void __launch_bounds__(kRowThreads) xent_kernel(const float* __restrict__ logits, T* dlogits,
                                                           const int32_t* __restrict__ tok, int s, int V,
                                                           float scale, double* loss_sum) {
  __shared__ float red_m[8], red_z[8];
  const long long row = blockIdx.x;
  const int bi = (int)(row / s), t = (int)(row % s);
  const int target = tok[bi * (s + 1) + t + 1];
  const float* lr = logits + row * V;
  T* dr = dlogits + row * V;
  const bool vec = (V & 3) == 0;
  const int V4 = vec ? V / 4 : 0;
  const float4* l4 = reinterpret_cast<const float4*>(lr);
  float m = -INFINITY, z = 0.0f;
  for (int v = threadIdx.x; v < V4; v += kRowThreads) {
    const float4 x = l4[v];
    const float mx = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
    if (mx > m) {
      z *= __expf(m - mx);
      m = mx;
    }
    z += __expf(x.x - m) + __expf(x.y - m) + __expf(x.z - m) + __expf(x.w - m);
  }
  for (int v = 4 * V4 + threadIdx.x; v < V; v += kRowThreads) online_add(m, z, lr[v]);
  // combine (m, z) pairs: warp shuffles, then the 8 warps through shared memory
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o), zo = __shfl_xor_sync(0xffffffffu, z, o);
    const float mn = fmaxf(m, mo);
    z = (m == -INFINITY ? 0.0f : z * __expf(m - mn)) + (mo == -INFINITY ? 0.0f : zo * __expf(mo - mn));
    m = mn;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red_m[w] = m;
    red_z[w] = z;
  }
  __syncthreads();
  float M = -INFINITY;
  for (int i = 0; i < kRowThreads / 32; ++i) M = fmaxf(M, red_m[i]);
  float Z = 0.0f;
  for (int i = 0; i < kRowThreads / 32; ++i)
    if (red_m[i] != -INFINITY) Z += red_z[i] * __expf(red_m[i] - M);
  const float lse = M + logf(Z);
  for (int v = threadIdx.x; v < V4; v += kRowThreads) {
    const float4 x = l4[v];
    const int e = 4 * v;
    st4<T>(dr + e, (__expf(x.x - lse) - (e == target ? 1.0f : 0.0f)) * scale,
           (__expf(x.y - lse) - (e + 1 == target ? 1.0f : 0.0f)) * scale,
           (__expf(x.z - lse) - (e + 2 == target ? 1.0f : 0.0f)) * scale,
           (__expf(x.w - lse) - (e + 3 == target ? 1.0f : 0.0f)) * scale);
  }
  for (int v = 4 * V4 + threadIdx.x; v < V; v += kRowThreads)
    st(dr + v, (__expf(lr[v] - lse) - (v == target ? 1.0f : 0.0f)) * scale);
  if (threadIdx.x == 0) atomicAdd(loss_sum, (double)(lse - lr[target]));
}

__device__ __forceinline__ float adam_update(float& p, float& m, float& v, float g, float b1, float b2,
                                             float lr, float eps, float wd, float bc1, float bc2) {
  m = b1 * m + (1.0f - b1) * g;
  v = b2 * v + (1.0f - b2) * g * g;
  const float mh = m / bc1, vh = v / bc2;
  p = p - lr * (mh / (sqrtf(vh) + eps) + wd * p);
  return p;
}

struct AdamK {
  float b1, b2, lr, eps, wd, bc1, bc2, scale;
};

template <typename T>
__global__ void adam_kernel(AdamK k, float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ g, T* __restrict__ plp, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float p = master[i], mi = m[i], vi = v[i];
    adam_update(p, mi, vi, g[i] * k.scale, k.b1, k.b2, k.lr, k.eps, k.wd, k.bc1, k.bc2);
    master[i] = p;
    m[i] = mi;
    v[i] = vi;
    if (plp) st(plp + i, p);
  }
}

// Packed state [master, m, v] per element: each thread owns 4 consecutive
// elements = 48 bytes of state (3 x float4) + 16 bytes of gradient.
template <typename T>
__global__ void adam_packed_kernel(AdamK k, float* __restrict__ state, const float* __restrict__ g,
                                   T* __restrict__ plp, long long n) {
  const long long n4 = n / 4;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x) {
    float4* s4 = reinterpret_cast<float4*>(state + q * 12);
    float4 a = s4[0], b = s4[1], c = s4[2];
    const float4 gg = reinterpret_cast<const float4*>(g)[q];
    float e[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    const float gv[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      adam_update(e[3 * j], e[3 * j + 1], e[3 * j + 2], gv[j] * k.scale, k.b1, k.b2, k.lr, k.eps, k.wd, k.bc1, k.bc2);
      if (plp) st(plp + q * 4 + j, e[3 * j]);
    }
    s4[0] = make_float4(e[0], e[1], e[2], e[3]);
    s4[1] = make_float4(e[4], e[5], e[6], e[7]);
    s4[2] = make_float4(e[8], e[9], e[10], e[11]);
  }
  // tail (n % 4) handled by block 0
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const long long i = n4 * 4 + threadIdx.x;
    float* e = state + i * 3;
    adam_update(e[0], e[1], e[2], g[i] * k.scale, k.b1, k.b2, k.lr, k.eps, k.wd, k.bc1, k.bc2);
    if (plp) st(plp + i, e[0]);
  }
}

template <typename T>
__global__ void cast_kernel(const float* __restrict__ src, T* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    st(dst + i, src[i]);
}

AdamK make_adam(const AdamHyper& hp, int step, float scale) {
  AdamK k;
  k.b1 = hp.beta1;
  k.b2 = hp.beta2;
  k.lr = hp.lr;
  k.eps = hp.eps;
  k.wd = hp.weight_decay;
  k.bc1 = (float)(1.0 - std::pow((double)hp.beta1, step));
  k.bc2 = (float)(1.0 - std::pow((double)hp.beta2, step));
  k.scale = scale;
  return k;
}

using bf16 = __nv_bfloat16;

#define GS_DISPATCH(dt, ...)                 \
  do {                                       \
    if ((dt) == DType::F32) {                \
      using T = float;                       \
      __VA_ARGS__;                           \
    } else {                                 \
      using T = bf16;                        \
      __VA_ARGS__;                           \
    }                                        \
  } while (0)

}  // namespace

cudaError_t layernorm_fwd(DType dt, const void* x, void* y, float* mean, float* rstd, int rows, int h,
                          cudaStream_t s) {
  if (h > kRowThreads * kMaxPerThread) return cudaErrorInvalidValue;
  if (rows == 0) return cudaSuccess;
  GS_DISPATCH(dt, {
    if (h % Vec<T>::N == 0) {
      const RowShape r = row_shape(h, Vec<T>::N, 4);
      GS_ROW_C(r.c, GS_TRY_E(launch_pdl(ln_fwd_vec_kernel<T, C>, dim3((rows + r.rpb - 1) / r.rpb),
                                        dim3(32 * r.nw * r.rpb), 0, s, (const T*)x, (T*)y, mean, rstd, rows, h, r.nw)));
    } else {
      GS_ROW_E(h, ln_fwd_kernel<T, E><<<rows, kRowThreads, 0, s>>>((const T*)x, (T*)y, mean, rstd, h));
    }
  });
  count_launch();
  return cudaGetLastError();
}

cudaError_t layernorm_bwd(DType dt, const void* x, const float* mean, const float* rstd, const void* dy,
                          const void* res, void* dx, int rows, int h, cudaStream_t s) {
  if (h > kRowThreads * kMaxPerThread) return cudaErrorInvalidValue;
  if (rows == 0) return cudaSuccess;
  GS_DISPATCH(dt, {
    if (h % Vec<T>::N == 0) {
      const RowShape r = row_shape(h, Vec<T>::N, 2);
      GS_ROW_C(r.c, GS_TRY_E(launch_pdl(ln_bwd_vec_kernel<T, C>, dim3((rows + r.rpb - 1) / r.rpb),
                                        dim3(32 * r.nw * r.rpb), 0, s, (const T*)x, mean, rstd, (const T*)dy,
                                        (const T*)res, (T*)dx, rows, h, r.nw)));
    } else {
      if (res && res != dx) {
        cudaError_t e = cudaMemcpyAsync(dx, res, (size_t)rows * h * sizeof(T), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
      }
      GS_ROW_E(h, ln_bwd_kernel<T, E><<<rows, kRowThreads, 0, s>>>((const T*)x, mean, rstd, (const T*)dy, (T*)dx,
                                                                   h, res != nullptr));
    }
  });
  count_launch();
  return cudaGetLastError();
}

cudaError_t gelu_fwd(DType dt, const void* u, void* g, long long n, cudaStream_t s) {
  GS_DISPATCH(dt, gelu_fwd_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>((const T*)u, (T*)g, n));
  count_launch();
  return cudaGetLastError();
}
cudaError_t gelu_bwd(DType dt, const void* u, const void* dg, void* du, long long n, cudaStream_t s) {
  GS_DISPATCH(dt, gelu_bwd_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>((const T*)u, (const T*)dg, (T*)du, n));
  count_launch();
  return cudaGetLastError();
}
cudaError_t add(DType dt, const void* a, const void* b, void* y, long long n, cudaStream_t s) {
  GS_DISPATCH(dt, add_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>((const T*)a, (const T*)b, (T*)y, n));
  count_launch();
  return cudaGetLastError();
}
cudaError_t fill_zero(void* p, size_t bytes, cudaStream_t s) { return cudaMemsetAsync(p, 0, bytes, s); }

// One-CTA no-op grid launched without the programmatic-serialisation
// attribute: it starts only once its predecessor grid has fully completed and
// never triggers its dependents early, so a CUDA event recorded after it
// marks that completion (the profiler's fence around a timed launch).
__global__ void stream_fence_kernel() {}
cudaError_t stream_fence(cudaStream_t s) {
  stream_fence_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

__global__ void copy_words_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
cudaError_t copy_words(uint32_t* dst, const uint32_t* src, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  copy_words_kernel<<<grid_for(n, 256), 256, 0, s>>>(dst, src, n);
  count_launch();
  return cudaGetLastError();
}

// Token ids of an iteration: copied (src may be mapped pinned host memory),
// range-checked against the vocabulary.  An id outside [0, V) would index
// past wte / dwte in the embedding, head and loss kernels: it is replaced by
// 0 and counted in *bad, which the executor checks after the run.
__global__ void copy_tokens_kernel(int32_t* __restrict__ dst, const int32_t* __restrict__ src, long long n, int V,
                                   int* __restrict__ bad) {
  int nbad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int32_t t = src[i];
    if (t < 0 || t >= V) {
      t = 0;
      ++nbad;
    }
    dst[i] = t;
  }
  if (nbad) atomicAdd(bad, nbad);
}
cudaError_t copy_tokens(int32_t* dst, const int32_t* src, long long n, int vocab, int* bad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  copy_tokens_kernel<<<grid_for(n, 256), 256, 0, s>>>(dst, src, n, vocab, bad);
  count_launch();
  return cudaGetLastError();
}

cudaError_t embed_fwd(DType dt, const void* wte, const void* wpe, const int32_t* tok, void* x0, int b, int s,
                      int h, cudaStream_t st) {
  GS_DISPATCH(dt, embed_fwd_kernel<T><<<b * s, 256, 0, st>>>((const T*)wte, (const T*)wpe, tok, (T*)x0, s, h));
  count_launch();
  return cudaGetLastError();
}
cudaError_t embed_bwd(DType dt, const int32_t* tok, const void* dx0, float* dwte, float* dwpe, int b, int s,
                      int h, cudaStream_t st) {
  GS_DISPATCH(dt, embed_bwd_kernel<T><<<b * s, 256, 0, st>>>(tok, (const T*)dx0, dwte, dwpe, s, h));
  count_launch();
  return cudaGetLastError();
}
cudaError_t softmax_xent(const float* logits, void* dlogits, DType dt, const int32_t* tok, int b, int s, int V,
                         float scale, double* loss_sum, cudaStream_t st) {
  GS_DISPATCH(dt, xent_kernel<T><<<b * s, kRowThreads, 0, st>>>(logits, (T*)dlogits, tok, s, V, scale, loss_sum));
  count_launch();
  return cudaGetLastError();
}

cudaError_t adam_step(const AdamHyper& hp, int step, float grad_scale, float* master, float* m, float* v,
                      const float* grad, void* param_lp, DType lp_dt, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const AdamK k = make_adam(hp, step, grad_scale);
  GS_DISPATCH(lp_dt, adam_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>(k, master, m, v, grad, (T*)param_lp, n));
  count_launch();
  return cudaGetLastError();
}

cudaError_t adam_step_packed(const AdamHyper& hp, int step, float grad_scale, float* state, const float* grad,
                             void* param_lp, DType lp_dt, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // float4 paths need 16-byte aligned state/grad; callers pass chunk starts
  // that are multiples of 4 elements.
  if ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(grad)) & 15) return cudaErrorMisalignedAddress;
  const AdamK k = make_adam(hp, step, grad_scale);
  GS_DISPATCH(lp_dt, adam_packed_kernel<T><<<grid_for(n / 4 + 1, 256, 2), 256, 0, s>>>(k, state, grad, (T*)param_lp, n));
  count_launch();
  return cudaGetLastError();
}

cudaError_t cast_from_f32(DType dt, const float* src, void* dst, long long n, cudaStream_t s) {
  GS_DISPATCH(dt, cast_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>(src, (T*)dst, n));
  count_launch();
  return cudaGetLastError();
}

}  // namespace gs

namespace gs {
long long& launch_counter_ref() {
  static long long n = 0;
  return n;
}
}  // namespace gs
