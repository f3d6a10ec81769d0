// Host-core Adam (engine/host_adam.cpp, the AVX-512 path and its scalar
// tail) against a plain restatement of the same arithmetic — the update of
// gso_adam_step (oracle/gs_oracle.c) with the FMA contraction the compiled
// loops use — on 3,000,007 elements: every fp32 state word and bf16 output
// must be bit-identical.  Built and run by tests/test_host_adam.py (CPU).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "host_adam.hpp"

using namespace gs::engine;

static uint16_t rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}

int main() {
  const uint64_t n = 3000007;
  std::mt19937 r(1);
  std::normal_distribution<float> N(0, 1);
  std::vector<float> st(3 * n), g(n);
  for (auto& x : st) x = N(r) * 0.02f;
  for (uint64_t i = 0; i < n; ++i) {
    st[3 * i + 2] = std::fabs(st[3 * i + 2]) * 0.01f;
    g[i] = N(r) * 0.01f;
  }
  const HostAdamHyper hp{1e-3f, 0.9f, 0.95f, 1e-8f, 0.01f};
  const int step = 3;
  const float bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(hp.beta1), step));
  const float bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(hp.beta2), step));
  std::vector<float> ref = st;
  std::vector<uint16_t> ref_lp(n);
  std::vector<float> ref_f32(n);
  for (uint64_t i = 0; i < n; ++i) {
    float* s = &ref[3 * i];
    const float m = std::fma(hp.beta1, s[1], (1.0f - hp.beta1) * g[i]);
    const float v = std::fma(hp.beta2, s[2], ((1.0f - hp.beta2) * g[i]) * g[i]);
    const float mh = m / bc1, vh = v / bc2;
    const float p = std::fma(-hp.lr, std::fma(hp.weight_decay, s[0], mh / (std::sqrt(vh) + hp.eps)), s[0]);
    s[0] = p;
    s[1] = m;
    s[2] = v;
    ref_lp[i] = rne(p);
    ref_f32[i] = p;
  }
  int fails = 0;
  for (int lp : {2, 4}) {
    ThreadPool pool(4, 0);
    std::vector<float> a = st;
    std::vector<uint16_t> o16(n);
    std::vector<float> o32(n);
    host_adam_step(hp, step, a.data(), g.data(), lp == 2 ? static_cast<void*>(o16.data()) : o32.data(), lp, n, pool);
    uint64_t bad = 0;
    for (uint64_t i = 0; i < 3 * n; ++i) bad += std::memcmp(&a[i], &ref[i], 4) != 0;
    for (uint64_t i = 0; i < n; ++i)
      bad += lp == 2 ? (o16[i] != ref_lp[i]) : (std::memcmp(&o32[i], &ref_f32[i], 4) != 0);
    std::printf("lp=%d: %llu differing words\n", lp, static_cast<unsigned long long>(bad));
    fails += bad != 0;
  }
  return fails;
}
