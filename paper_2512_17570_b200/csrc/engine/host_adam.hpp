// CpuStep on the host cores: the reference's optimizer placement
// (proj/src/simulator.cpp:24-43 charges CpuStep to the CPU resource at
// MachineSpec::cpu_step_throughput; PAPER.md:571-584 — fp32 master, m, v in
// CPU memory, gradients offloaded by the GradAccum D2H, the updated
// low-precision parameters written straight into their CPU-resident copy).
#pragma once

#include <cstdint>

#include "host_tiers.hpp"

namespace gs::engine {

struct HostAdamHyper {
  float lr, beta1, beta2, eps, weight_decay;
};

// Adam over n elements: state is packed [master, m, v] per element (the
// executor's optimizer-state layout), grad fp32, lp_out bf16 (lp_bytes 2) or
// fp32 (4).  Same arithmetic as the GPU kernel (kernels/elementwise.cu
// adam_update) and the oracle (gso_adam_step).  Split over the pool's
// threads in cache-line-aligned blocks; AVX-512 where the CPU has it
// (bit-identical to the scalar loop, tests/test_host_adam.py).
void host_adam_step(const HostAdamHyper& hp, int step, float* state, const float* grad, void* lp_out, int lp_bytes,
                    uint64_t n, ThreadPool& pool);

}  // namespace gs::engine
