// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cstdlib>
#include <utility>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gs {

// Storage types of the two precision modes: fp32 parity mode
// (ModelSpec.low_precision_bytes = 4) and bf16 training mode (= 2).
template <typename T> struct io;
template <> struct io<float> {
  __device__ __forceinline__ static float load(const float* p) { return *p; }
  __device__ __forceinline__ static void store(float* p, float v) { *p = v; }
};
template <> struct io<__nv_bfloat16> {
  __device__ __forceinline__ static float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};
template <typename T> __device__ __forceinline__ float ld(const T* p) { return io<T>::load(p); }
template <typename T> __device__ __forceinline__ void st(T* p, float v) { io<T>::store(p, v); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// tanh-approximation GELU (matches torch gelu(approximate="tanh")).
constexpr float kGeluK = 0.7978845608028654f;
constexpr float kGeluC = 0.044715f;
__device__ __forceinline__ float gelu_f(float u) {
  return 0.5f * u * (1.0f + tanhf(kGeluK * (u + kGeluC * u * u * u)));
}
__device__ __forceinline__ float gelu_grad_f(float u) {
  const float t = tanhf(kGeluK * (u + kGeluC * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * kGeluK * (1.0f + 3.0f * kGeluC * u * u);
}

// bf16-path variants on the SFU tanh (tanh.approx.f32, |rel err| < 2^-10.9):
// the result is rounded to bf16 (2^-8) right after, so the accurate libm
// tanhf (~20 FP32 instructions) only costs GEMM-epilogue issue slots.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float u) {
  return 0.5f * u * (1.0f + tanh_fast(kGeluK * (u + kGeluC * u * u * u)));
}
__device__ __forceinline__ float gelu_grad_fast(float u) {
  const float t = tanh_fast(kGeluK * (u + kGeluC * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * kGeluK * (1.0f + 3.0f * kGeluC * u * u);
}

// Kernels launched through this library (host-side count, all threads).
long long& launch_counter_ref();
inline void count_launch(int n = 1) { __atomic_fetch_add(&launch_counter_ref(), (long long)n, __ATOMIC_RELAXED); }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Programmatic dependent launch (PDL): kernels on the layer chain are
// launched with programmatic stream serialisation and open with
// pdl_trigger_and_wait(): the next kernel's CTAs may be scheduled while this
// grid's last CTAs run, but no CTA touches memory before its predecessor grid
// has completed (griddepcontrol.wait), so stream order semantics are kept.
// griddepcontrol.* are no-ops for a kernel launched without the attribute.
// The wait comes first in every kernel, before TMEM allocation too: a
// dependent CTA that allocated TMEM before its wait could starve a primary
// CTA that has triggered but not yet allocated (measured: an 85k-token/s
// outlier run with the wait moved after the allocation).
// GS_PDL=0 launches without it.
__device__ __forceinline__ void pdl_trigger_and_wait() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GS_PDL");
    return !e || atoi(e) != 0;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline unsigned grid_for(long long n, int block, int per_thread = 1) {
  long long g = (n + (long long)block * per_thread - 1) / ((long long)block * per_thread);
  const long long cap = 32LL * num_sms();
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace gs
