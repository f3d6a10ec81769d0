// CUDA-core tiled GEMM: the fp32 parity-mode path (ModelSpec.low_precision_
// bytes = 4, where tensor-core rounding would break the 1e-4 parameter
// tolerance) and the fallback for shapes the tcgen05 kernel does not tile.
// 64x64 output tile per 256-thread CTA, 4x4 outputs per thread, BK=16 staged
// through shared memory, fp32 accumulation, fused epilogues (residual add,
// GELU, fp32 gradient accumulation).
#include "common.cuh"
#include "kernels.h"

namespace gs {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;

template <typename T, bool AK, bool BKM, int EPI>
__global__ void __launch_bounds__(256) simt_gemm_kernel(int M, int N, int K, const T* __restrict__ A,
                                                        const T* __restrict__ B, void* C, const T* R, T* G,
                                                        int ldc) {
  __shared__ float As[BK][BM + PAD];
  __shared__ float Bs[BK][BN + PAD];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tr = tid / 16, tc = tid % 16;  // 16x16 threads, 4x4 outputs each
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    // each thread loads 4 elements of A-tile and 4 of B-tile
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int idx = tid + r * 256;  // 0..1023 over a 64x16 tile
      int mm, kk;
      if (AK) { mm = idx / BK; kk = idx % BK; } else { kk = idx / BM; mm = idx % BM; }
      const int gm = m0 + mm, gk = k0 + kk;
      float av = 0.0f;
      if (gm < M && gk < K) av = ld(AK ? A + (long long)gm * K + gk : A + (long long)gk * M + gm);
      As[kk][mm] = av;
      int nn, kb;
      if (BKM) { nn = idx / BK; kb = idx % BK; } else { kb = idx / BN; nn = idx % BN; }
      const int gn = n0 + nn, gkb = k0 + kb;
      float bv = 0.0f;
      if (gn < N && gkb < K) bv = ld(BKM ? B + (long long)gn * K + gkb : B + (long long)gkb * N + gn);
      Bs[kb][nn] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tc + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + tr + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tc + 16 * j;
      if (gn >= N) continue;
      const long long o = (long long)gm * ldc + gn;
      const float v = acc[i][j];
      if (EPI == (int)Epi::Store) st((T*)C + o, v);
      else if (EPI == (int)Epi::AddResidual) st((T*)C + o, v + ld(R + o));
      else if (EPI == (int)Epi::AccumF32) ((float*)C)[o] += v;
      else if (EPI == (int)Epi::StoreGelu) { st((T*)C + o, v); st(G + o, gelu_f(ld((T*)C + o))); }
      else if (EPI == (int)Epi::MulGeluGrad) { st((T*)C + o, v); st((T*)C + o, ld((T*)C + o) * gelu_grad_f(ld(R + o))); }
      else if (EPI == (int)Epi::Gelu) { st((T*)C + o, v); st((T*)C + o, gelu_f(ld((T*)C + o))); }
      else ((float*)C)[o] = v;
    }
  }
}

template <typename T, bool AK, bool BKM>
cudaError_t launch_epi(const GemmArgs& g, cudaStream_t s) {
  const dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM);
  const int ldc = g.ldc ? g.ldc : g.N;
  const T* A = (const T*)g.A;
  const T* B = (const T*)g.B;
  count_launch();
  switch (g.epi) {
    case Epi::Store: simt_gemm_kernel<T, AK, BKM, 0><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::AddResidual: simt_gemm_kernel<T, AK, BKM, 1><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::AccumF32: simt_gemm_kernel<T, AK, BKM, 2><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::StoreGelu: simt_gemm_kernel<T, AK, BKM, 3><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::StoreF32: simt_gemm_kernel<T, AK, BKM, 4><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::MulGeluGrad: simt_gemm_kernel<T, AK, BKM, 5><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
    case Epi::Gelu: simt_gemm_kernel<T, AK, BKM, 6><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, B, g.C, (const T*)g.R, (T*)g.G, ldc); break;
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t s) {
  if (g.a_kmajor && g.b_kmajor) return launch_epi<T, true, true>(g, s);
  if (g.a_kmajor && !g.b_kmajor) return launch_epi<T, true, false>(g, s);
  if (!g.a_kmajor && g.b_kmajor) return launch_epi<T, false, true>(g, s);
  return launch_epi<T, false, false>(g, s);
}

}  // namespace

cudaError_t gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.K <= 0) return cudaErrorInvalidValue;
  return g.dt == DType::F32 ? launch_t<float>(g, s) : launch_t<__nv_bfloat16>(g, s);
}

cudaError_t gemm(const GemmArgs& g, cudaStream_t s) {
  if (gemm_tc_supported(g)) return gemm_tc(g, s);
  return gemm_simt(g, s);
}

}  // namespace gs
