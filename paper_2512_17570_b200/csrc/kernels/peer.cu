// Data-parallel reduction over peer memory (engine/peer_comm.hpp): each rank
// reads every rank's fp32 partial of its own shard straight out of the
// peers' HBM (CUDA IPC mappings; NVLink 5 / NVSwitch loads on a multi-GPU
// node, plain HBM loads for ranks sharing a device) and writes the sum.
// Sums run in rank order, so every rank's shard is bit-identical to a
// single-process sum in that order, run after run.  NVLink / HBM bound:
// float4 loads from every rank per thread, a capped grid (32 CTAs) so the
// reduce leaves the SMs to the compute stream it overlaps.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace gs {

namespace {

template <int W>
__global__ void __launch_bounds__(256) peer_sum_kernel(PeerSrcs src, float* __restrict__ dst, long long n) {
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 acc = __ldcg(reinterpret_cast<const float4*>(src.p[0]) + i);
#pragma unroll
    for (int r = 1; r < W; ++r) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src.p[r]) + i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(dst)[i] = acc;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    float acc = __ldcg(src.p[0] + i);
#pragma unroll
    for (int r = 1; r < W; ++r) acc += __ldcg(src.p[r] + i);
    dst[i] = acc;
  }
}

// One thread: make every prior write of this stream visible system-wide,
// then publish `value` into each rank's counter with a release store (the
// counters of the other ranks are IPC mappings of their device memory).
__global__ void peer_signal_kernel(PeerFlags f, int n, uint32_t value) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int r = 0; r < n; ++r) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[r]), "r"(value) : "memory");
}

// Fallback wait (devices without stream wait-value support): one thread
// spins with acquire loads until every counter reaches `value`.
__global__ void peer_wait_kernel(PeerFlags f, int n, uint32_t value) {
  if (threadIdx.x != 0) return;
  for (int r = 0; r < n; ++r) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f.p[r]) : "memory");
    } while (static_cast<int32_t>(v - value) < 0);
  }
}

}  // namespace

cudaError_t peer_signal(const PeerFlags& f, int n, uint32_t value, cudaStream_t s) {
  if (n < 0 || n > kMaxPeers) return cudaErrorInvalidValue;
  count_launch();
  peer_signal_kernel<<<1, 32, 0, s>>>(f, n, value);
  return cudaGetLastError();
}

cudaError_t peer_wait_spin(const PeerFlags& f, int n, uint32_t value, cudaStream_t s) {
  if (n < 0 || n > kMaxPeers) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  count_launch();
  peer_wait_kernel<<<1, 32, 0, s>>>(f, n, value);
  return cudaGetLastError();
}

cudaError_t peer_sum(const PeerSrcs& src, int world, float* dst, long long n, cudaStream_t s) {
  if (world < 1 || world > kMaxPeers || n < 0) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  // a few CTAs saturate the peer links (each thread keeps W 16-byte loads in
  // flight); the reduce runs beside the next stage's GEMMs, so it must not
  // take their SMs (a 32-per-SM grid would)
  const unsigned grid = std::min(grid_for(n / 4 + 1, 256), 32u);
  count_launch();
  switch (world) {
    case 1: peer_sum_kernel<1><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 2: peer_sum_kernel<2><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 3: peer_sum_kernel<3><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 4: peer_sum_kernel<4><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 5: peer_sum_kernel<5><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 6: peer_sum_kernel<6><<<grid, 256, 0, s>>>(src, dst, n); break;
    case 7: peer_sum_kernel<7><<<grid, 256, 0, s>>>(src, dst, n); break;
    default: peer_sum_kernel<8><<<grid, 256, 0, s>>>(src, dst, n); break;
  }
  return cudaGetLastError();
}

}  // namespace gs
