#include "host_adam.hpp"

#include <immintrin.h>

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

// AVX-512 form of run_range: 16 elements per step, the AoS state
// de-interleaved with two-source permutes, the same operations in the same
// order as the scalar loop (IEEE div / sqrt, so the results are identical),
// bf16 by the same round-to-nearest-even on the integer bits.  The scalar
// loop compiled to scalar vdivss / vsqrtss (the stride-3 AoS access defeats
// the auto-vectoriser), ~3 Gelem/s on the GPU box's 16 cores; this form is
// DRAM-bound.
struct Lanes {
  __m512i src01[3], src2[3];  // de-interleave: component c of elements 0..15
  __mmask16 hi[3];            // lanes whose source index is >= 32 (in the third vector)
  __m512i dst01[3], dst2[3];  // re-interleave: output vector q, lanes from (p, m) / v
  __mmask16 from_v[3];
};

__attribute__((target("avx512f"))) Lanes make_lanes() {
  Lanes L;
  alignas(64) int a[16], b[16];
  for (int c = 0; c < 3; ++c) {
    unsigned hm = 0;
    for (int j = 0; j < 16; ++j) {
      const int src = 3 * j + c;
      a[j] = src < 32 ? src : 0;
      b[j] = src >= 32 ? src - 32 : 0;
      if (src >= 32) hm |= 1u << j;
    }
    L.src01[c] = _mm512_load_si512(a);
    L.src2[c] = _mm512_load_si512(b);
    L.hi[c] = static_cast<__mmask16>(hm);
  }
  // output vector q holds AoS positions 16q .. 16q+15: element e = pos / 3,
  // component c = pos % 3; p / m come from permutex2var(p, idx, m) (m lanes
  // offset by 16), v from a masked permutexvar
  for (int q = 0; q < 3; ++q) {
    unsigned vm = 0;
    for (int i = 0; i < 16; ++i) {
      const int pos = 16 * q + i, e = pos / 3, c = pos % 3;
      a[i] = c == 0 ? e : (c == 1 ? 16 + e : 0);
      b[i] = c == 2 ? e : 0;
      if (c == 2) vm |= 1u << i;
    }
    L.dst01[q] = _mm512_load_si512(a);
    L.dst2[q] = _mm512_load_si512(b);
    L.from_v[q] = static_cast<__mmask16>(vm);
  }
  return L;
}

template <int LP>
__attribute__((target("avx512f"))) uint64_t run_range_avx512(const K& k, float* __restrict__ st,
                                                             const float* __restrict__ g, void* __restrict__ out,
                                                             uint64_t lo, uint64_t hi) {
  static const Lanes L = make_lanes();
  const __m512 b1 = _mm512_set1_ps(k.b1), b2 = _mm512_set1_ps(k.b2);
  const __m512 ob1 = _mm512_set1_ps(1.0f - k.b1), ob2 = _mm512_set1_ps(1.0f - k.b2);
  const __m512 bc1 = _mm512_set1_ps(k.bc1), bc2 = _mm512_set1_ps(k.bc2);
  const __m512 lr = _mm512_set1_ps(k.lr), eps = _mm512_set1_ps(k.eps), wd = _mm512_set1_ps(k.wd);
  uint64_t i = lo;
  for (; i + 16 <= hi; i += 16) {
    float* s = st + 3 * i;
    const __m512 a0 = _mm512_loadu_ps(s), a1 = _mm512_loadu_ps(s + 16), a2 = _mm512_loadu_ps(s + 32);
    __m512 c3[3];
    for (int c = 0; c < 3; ++c)
      c3[c] = _mm512_mask_permutexvar_ps(_mm512_permutex2var_ps(a0, L.src01[c], a1), L.hi[c], L.src2[c], a2);
    __m512 p = c3[0], m = c3[1], v = c3[2];
    const __m512 gg = _mm512_loadu_ps(g + i);
    // scalar: m = b1*m + (1-b1)*g, v = b2*v + (1-b2)*g*g (contracted to FMA
    // by the compiler the same way: fma(b1, m, (1-b1)*g))
    m = _mm512_fmadd_ps(b1, m, _mm512_mul_ps(ob1, gg));
    v = _mm512_fmadd_ps(b2, v, _mm512_mul_ps(_mm512_mul_ps(ob2, gg), gg));
    const __m512 mh = _mm512_div_ps(m, bc1), vh = _mm512_div_ps(v, bc2);
    const __m512 upd = _mm512_fmadd_ps(wd, p, _mm512_div_ps(mh, _mm512_add_ps(_mm512_sqrt_ps(vh), eps)));
    p = _mm512_fnmadd_ps(lr, upd, p);
    for (int q = 0; q < 3; ++q)
      _mm512_storeu_ps(s + 16 * q,
                       _mm512_mask_permutexvar_ps(_mm512_permutex2var_ps(p, L.dst01[q], m), L.from_v[q], L.dst2[q], v));
    if constexpr (LP == 2) {
      __m512i u = _mm512_castps_si512(p);
      const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(u, 16), _mm512_set1_epi32(1));
      u = _mm512_add_epi32(u, _mm512_add_epi32(_mm512_set1_epi32(0x7FFF), lsb));
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(static_cast<uint16_t*>(out) + i),
                          _mm512_cvtepi32_epi16(_mm512_srli_epi32(u, 16)));
    } else {
      _mm512_storeu_ps(static_cast<float*>(out) + i, p);
    }
  }
  return i;
}

bool have_avx512() {
  static const bool yes = __builtin_cpu_supports("avx512f");
  return yes;
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
      jobs.emplace_back([=, &k] {
        const uint64_t done = have_avx512() ? run_range_avx512<2>(k, state, grad, lp_out, lo, hi) : lo;
        run_range<2>(k, state, grad, lp_out, done, hi);
      });
    else
      jobs.emplace_back([=, &k] {
        const uint64_t done = have_avx512() ? run_range_avx512<4>(k, state, grad, lp_out, lo, hi) : lo;
        run_range<4>(k, state, grad, lp_out, done, hi);
      });
  }
  pool.run_all(jobs);
}

}  // namespace gs::engine
