#include "host_adam.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

namespace gs::engine {

namespace {

inline uint16_t bf16_rne(float f) {  // round to nearest even (finite inputs)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}

struct K {
  float b1, b2, lr, eps, wd, bc1, bc2;
};

// 16 elements at a time: de-interleave the packed state into lanes, update,
// re-interleave (the lane loops vectorise; the pass is DRAM-bound at
// 30 B/element).
template <int LP>
void run_range(const K& k, float* __restrict__ st, const float* __restrict__ g, void* __restrict__ out, uint64_t lo,
               uint64_t hi) {
  constexpr int B = 16;
  uint64_t i = lo;
  for (; i + B <= hi; i += B) {
    float p[B], m[B], v[B], gg[B];
    float* s = st + 3 * i;
    for (int j = 0; j < B; ++j) {
      p[j] = s[3 * j];
      m[j] = s[3 * j + 1];
      v[j] = s[3 * j + 2];
      gg[j] = g[i + j];
    }
    for (int j = 0; j < B; ++j) {
      m[j] = k.b1 * m[j] + (1.0f - k.b1) * gg[j];
      v[j] = k.b2 * v[j] + (1.0f - k.b2) * gg[j] * gg[j];
      const float mh = m[j] / k.bc1, vh = v[j] / k.bc2;
      p[j] = p[j] - k.lr * (mh / (std::sqrt(vh) + k.eps) + k.wd * p[j]);
    }
    for (int j = 0; j < B; ++j) {
      s[3 * j] = p[j];
      s[3 * j + 1] = m[j];
      s[3 * j + 2] = v[j];
    }
    if constexpr (LP == 2) {
      uint16_t* o = static_cast<uint16_t*>(out) + i;
      for (int j = 0; j < B; ++j) o[j] = bf16_rne(p[j]);
    } else {
      std::memcpy(static_cast<float*>(out) + i, p, sizeof p);
    }
  }
  for (; i < hi; ++i) {
    float* s = st + 3 * i;
    float m = k.b1 * s[1] + (1.0f - k.b1) * g[i];
    float v = k.b2 * s[2] + (1.0f - k.b2) * g[i] * g[i];
    const float mh = m / k.bc1, vh = v / k.bc2;
    const float p = s[0] - k.lr * (mh / (std::sqrt(vh) + k.eps) + k.wd * s[0]);
    s[0] = p;
    s[1] = m;
    s[2] = v;
    if constexpr (LP == 2) static_cast<uint16_t*>(out)[i] = bf16_rne(p);
    else static_cast<float*>(out)[i] = p;
  }
}

}  // namespace

void host_adam_step(const HostAdamHyper& hp, int step, float* state, const float* grad, void* lp_out, int lp_bytes,
                    uint64_t n, ThreadPool& pool) {
  if (n == 0) return;
  K k{hp.beta1, hp.beta2, hp.lr, hp.eps, hp.weight_decay,
      static_cast<float>(1.0 - std::pow(static_cast<double>(hp.beta1), step)),
      static_cast<float>(1.0 - std::pow(static_cast<double>(hp.beta2), step))};
  // ~4 blocks per thread keeps the pool busy when block times differ; block
  // bounds are multiples of 64 elements (whole cache lines of grad / state)
  const uint64_t parts = static_cast<uint64_t>(std::max(1, pool.size())) * 4;
  const uint64_t per = std::max<uint64_t>(1 << 14, (n + parts - 1) / parts + 63) / 64 * 64;
  std::vector<std::function<void()>> jobs;
  for (uint64_t lo = 0; lo < n; lo += per) {
    const uint64_t hi = std::min(n, lo + per);
    if (lp_bytes == 2)
      jobs.emplace_back([=, &k] { run_range<2>(k, state, grad, lp_out, lo, hi); });
    else
      jobs.emplace_back([=, &k] { run_range<4>(k, state, grad, lp_out, lo, hi); });
  }
  pool.run_all(jobs);
}

}  // namespace gs::engine
