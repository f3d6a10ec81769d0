// PCIe probe: SM-driven zero-copy reads / writes of mapped pinned host memory
// vs copy-engine DMA, alone and concurrently.  Diagnostics only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_probe zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    dst[i] = v;
  }
}
// 4 independent loads in flight per thread
__global__ void zc_read4(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * stride < n) v[k] = src[i + k * stride];
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * stride < n) dst[i + k * stride] = v[k];
  }
}

int main() {
  const size_t bytes = 1ull << 30, n = bytes / 16;
  void *h_a, *h_b, *d_a, *d_b;
  CK(cudaHostAlloc(&h_a, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_b, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d_a, bytes));
  CK(cudaMalloc(&d_b, bytes));
  memset(h_a, 1, bytes); memset(h_b, 2, bytes);
  void *m_a, *m_b;
  CK(cudaHostGetDevicePointer(&m_a, h_a, 0));
  CK(cudaHostGetDevicePointer(&m_b, h_b, 0));
  cudaStream_t s1, s2, s3;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double gb, auto&& f) {
    f(); cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(s1, e0); cudaStreamWaitEvent(s2, e0); cudaStreamWaitEvent(s3, e0);
    f();
    cudaEvent_t x1, x2, x3; cudaEventCreate(&x1); cudaEventCreate(&x2); cudaEventCreate(&x3);
    cudaEventRecord(x1, s1); cudaEventRecord(x2, s2); cudaEventRecord(x3, s3);
    cudaStreamWaitEvent(0, x1); cudaStreamWaitEvent(0, x2); cudaStreamWaitEvent(0, x3);
    cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\": \"%s\", \"ms\": %.2f, \"gb\": %.2f, \"gbs\": %.1f}\n", name, ms, gb, gb / (ms / 1e3));
  };
  const double G = bytes / 1e9;
  timeit("ce_h2d", G, [&] { cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s1); });
  timeit("ce_d2h", G, [&] { cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, s1); });
  timeit("ce_bidir(total)", 2 * G, [&] {
    cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, s2); });
  for (int ctas : {16, 32, 64, 148, 296}) {
    char nm[64];
    snprintf(nm, 64, "zc_read_ctas%d", ctas);
    timeit(nm, G, [&] { zc_read4<<<ctas, 512, 0, s1>>>((const uint4*)m_a, (uint4*)d_a, n); });
    snprintf(nm, 64, "zc_write_ctas%d", ctas);
    timeit(nm, G, [&] { zc_read4<<<ctas, 512, 0, s1>>>((const uint4*)d_b, (uint4*)m_b, n); });
    snprintf(nm, 64, "zc_readwrite_ctas%d(total)", ctas);
    timeit(nm, 2 * G, [&] { zc_read4<<<ctas, 512, 0, s1>>>((const uint4*)m_a, (uint4*)m_b, n); });
  }
  timeit("zc_read64+ce_h2d(total)", 2 * G, [&] {
    zc_read4<<<64, 512, 0, s1>>>((const uint4*)m_a, (uint4*)d_a, n);
    cudaMemcpyAsync(d_b, h_b, bytes, cudaMemcpyHostToDevice, s2); });
  timeit("ce_h2d_2streams(total)", 2 * G, [&] {
    cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(d_b, h_b, bytes, cudaMemcpyHostToDevice, s2); });
  return 0;
}
