// Causal attention forward on the 5th-generation tensor cores (sm_100a).
//
// One CTA per (128-query tile, batch x head), head_dim 128, bf16:
//   TMA (128B swizzle) loads Q once and K/V blocks of 128 keys into a
//   double-buffered ring; one elected thread issues
//     S_j = Q K_j^T      (tcgen05.mma kind::f16, M=128 N=128, fp32 in TMEM,
//                         two S buffers so S_{j+1} overlaps softmax_j)
//     O  += P_j V_j      (A = P from shared memory, B = V as an MN-major
//                         operand: no transpose)
//   four softmax warps own one query row (= one TMEM lane) each: tcgen05.ld
//   the S row, online softmax in registers (log2 domain), rescale O in TMEM
//   (tcgen05.ld / st) when the running max moves, write P in the UMMA
//   128B-swizzled K-major layout, and finally normalise O and write O / lse.
// Same layouts and semantics as the mma.sync path in attention.cu:
// qkv [b*s][3h] (q | k | v column blocks, head j at columns j*d),
// o [b*s][h], lse [b][H][s] natural log of the 1/sqrt(d)-scaled scores.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <climits>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace gs {

namespace {

using bf16 = __nv_bfloat16;

constexpr int kD = 128;       // head dim
constexpr int kBQ = 128;      // queries per CTA
constexpr int kBK = 128;      // keys per block
constexpr int kTile = kBQ * kD * 2;  // 32 KB: one 128 x 128 bf16 tile

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// A operand from tensor memory (TS form): A = [128 lanes][K] bf16 pairs
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// SWIZZLE_128B smem descriptor (sm_100 version bits).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// K-major 128 x 128 tile stored as two 64-wide swizzle chunks of 16 KB;
// k-step ks (16 elements) = chunk ks/4, +32 B inside the swizzle row.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int ks) {
  return sdesc(base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
}
// MN-major operand (V: keys x d with d contiguous): two 64-wide MN blocks of
// [128 k-rows][128 B] (LBO = 16 KB), 8-row K groups (SBO = 1 KB); k-step ks
// advances 16 rows.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int ks) {
  return sdesc(base + ks * 16 * 128, 16384, 1024);
}
constexpr uint32_t idesc(bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(128 >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

// SFU 2^x (ex2.approx.ftz: flushes denormal results; libm exp2f adds four
// range-fix instructions per element around the same MUFU op)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// GS_ATTN_TRACE grid schedule: {smid, start, end} of this CTA (see attn_trace_end)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cta_stamp(long long* tr, int slot) {
  if (!tr || threadIdx.x != 0) return;
  long long* c = tr + 8 * 64 + 4 * ((long long)blockIdx.y * gridDim.x + blockIdx.x);
  if (slot == 1) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    c[0] = sm;
  }
  c[slot] = gtimer();
}

// ------------------------------------------------------------ forward v3
// Two 128-query tiles per CTA and 128-key blocks, one CTA per SM (all 512
// TMEM columns: S0 | S1 | O0 | O1).  The S MMAs run at N = 128, where the
// SMEM operand stream (Q and K rows, 8 KB per 64-cycle MMA) keeps up with the
// tensor pipe — the N = 64 S MMAs of v2 run SMEM-bound — and the two tiles
// ping-pong: while softmax WG t works on S_t(kb+1), the pipe runs
// PV_{1-t}(kb) and S_{1-t}(kb+1).  P_t (bf16) is tcgen05.st-ed over S_t and
// O_t += P_t V is a TS-MMA.  Since each tile's S(kb) is issued after its
// PV(kb-1), seeing S_t(kb) means O_t is final for a rescale — no wait.
// 128 rows x 128 fp32 TMEM columns (lane = row, this warp's quarter) -> bf16
// (x scale) in shared memory as two SWIZZLE_128B boxes [2][128 rows][128 B],
// ready for store_tile_128.  Row-per-thread 16-byte stores, conflict-free
// under the swizzle.
__device__ __forceinline__ void stage_rows_bf16(uint32_t taddr, float scale, uint8_t* stg, int r) {
#pragma unroll
  for (int c = 0; c < kD / 32; ++c) {
    uint32_t rr[32];
    tld32(taddr + c * 32, rr);
    tld_wait();
    uint8_t* line = stg + (c >> 1) * 16384 + r * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = pack(__uint_as_float(rr[8 * q]) * scale, __uint_as_float(rr[8 * q + 1]) * scale);
      w.y = pack(__uint_as_float(rr[8 * q + 2]) * scale, __uint_as_float(rr[8 * q + 3]) * scale);
      w.z = pack(__uint_as_float(rr[8 * q + 4]) * scale, __uint_as_float(rr[8 * q + 5]) * scale);
      w.w = pack(__uint_as_float(rr[8 * q + 6]) * scale, __uint_as_float(rr[8 * q + 7]) * scale);
      *reinterpret_cast<uint4*>(line + ((((c & 1) * 4 + q) ^ (r & 7)) << 4)) = w;
    }
  }
}
// Two TMA stores (64 columns each) of a staged 128 x 128 bf16 tile at
// (col, row); waits until they are complete (the CTA may exit right after).
__device__ __forceinline__ void store_tile_128(const CUtensorMap* m, const uint8_t* stg, int col, int row) {
#pragma unroll
  for (int half = 0; half < 2; ++half)
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(su32(stg + half * 16384)), "r"(col + 64 * half), "r"(row)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr int kThreadsF3 = 320;  // w0 loads (thread 0), w1 MMA + TMEM, w2-5 / w6-9 softmax tiles 0 / 1
struct FaSmem3 {
  uint8_t Q[2][kTile];  // per tile: [2 d-chunks][128 rows][128 B]
  uint8_t K[2][kTile];  // 2-slot ring of 128-key blocks
  uint8_t V[2][kTile];
  // P_t is published in two halves (keys 0-63: p_lo, 64-127: p_hi) so the
  // first half of PV_t overlaps the softmax's second half
  uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_lo[2], p_hi[2], o_done[2];
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreadsF3, 1)
    fa_fwd_tc3_kernel(const __grid_constant__ CUtensorMap map_t, const __grid_constant__ CUtensorMap map_o,
                      bf16* __restrict__ o, float* __restrict__ lse, int s, int h, int H, float scale_log2,
                      long long* __restrict__ tr) {
  pdl_trigger_and_wait();
  extern __shared__ __align__(1024) uint8_t raw3[];
  FaSmem3& sm = *reinterpret_cast<FaSmem3*>(raw3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qp = gridDim.y - 1 - blockIdx.y;  // heaviest tile pairs first (LPT)
  const int bh = blockIdx.x, bi = bh / H, j = bh % H;
  const int row0 = bi * s, q0 = qp * 2 * kBQ;
  const int nblk0 = (q0 + kBQ) / kBK, nblk1 = nblk0 + 1;  // causal: tile t sees keys < q0 + 128 (t + 1)
  cta_stamp(tr, 1);
  if (threadIdx.x == 0) {
    bar_init(&sm.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      bar_init(&sm.k_full[i], 1);
      bar_init(&sm.k_empty[i], 1);
      bar_init(&sm.v_full[i], 1);
      bar_init(&sm.v_empty[i], 1);
      bar_init(&sm.s_full[i], 1);
      bar_init(&sm.p_lo[i], 128);
      bar_init(&sm.p_hi[i], 128);
      bar_init(&sm.o_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Thread 0 is the producer: Q of both tiles and the first K / V slots go
  // out before the CTA-wide sync, overlapping the TMEM allocation.
  auto load_k = [&](int kb) {
    const int sl = kb & 1;
    bar_expect(&sm.k_full[sl], kTile);
    for (int c = 0; c < 2; ++c)
      tma2d(sm.K[sl] + c * 16384, &map_t, &sm.k_full[sl], h + j * kD + 64 * c, row0 + kb * kBK);
  };
  auto load_v = [&](int kb) {
    const int sl = kb & 1;
    bar_expect(&sm.v_full[sl], kTile);
    for (int c = 0; c < 2; ++c)
      tma2d(sm.V[sl] + c * 16384, &map_t, &sm.v_full[sl], 2 * h + j * kD + 64 * c, row0 + kb * kBK);
  };
  const int n_early = nblk1 < 2 ? nblk1 : 2;  // ring slots that start empty
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_t)) : "memory");
    bar_expect(&sm.q_full, 2 * kTile);
    for (int t = 0; t < 2; ++t)
      for (int c = 0; c < 2; ++c)
        tma2d(sm.Q[t] + c * 16384, &map_t, &sm.q_full, j * kD + 64 * c, row0 + q0 + t * kBQ);
    for (int kb = 0; kb < n_early; ++kb) {
      load_k(kb);
      load_v(kb);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    if (lane == 0) {  // the rest of the K / V rings
      for (int kb = n_early; kb < nblk1; ++kb) {
        const int sl = kb & 1;
        bar_wait(&sm.k_empty[sl], ((kb >> 1) & 1) ^ 1);  // K(kb) after S_1(kb-2), not behind V's slot
        load_k(kb);
        bar_wait(&sm.v_empty[sl], ((kb >> 1) & 1) ^ 1);
        load_v(kb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      bar_wait(&sm.q_full, 0);
      auto issue_s = [&](int t, int kb) {  // S_t = Q_t K(kb)^T into columns [128 t, 128 t + 128)
        const uint32_t qa = su32(sm.Q[t]), ka = su32(sm.K[kb & 1]);
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks)
          mma(tmem + t * 128, desc_kmajor(qa, ks), desc_kmajor(ka, ks), idesc(false), ks != 0);
        commit(&sm.s_full[t]);
      };
      auto wait_k = [&](int kb) {
        bar_wait(&sm.k_full[kb & 1], (kb >> 1) & 1);
        fence_after();
      };
      auto issue_pv = [&](int t, int kb) {  // O_t += P_t V(kb), P_t from TMEM (8 columns per 16 keys)
        const uint32_t va = su32(sm.V[kb & 1]);
        bar_wait(&sm.p_lo[t], kb & 1);
        fence_after();
#pragma unroll
        for (int ks = 0; ks < kBK / 32; ++ks)
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + ks * 8, desc_mnmajor(va, ks), idesc(true), (kb | ks) != 0);
        bar_wait(&sm.p_hi[t], kb & 1);
        fence_after();
#pragma unroll
        for (int ks = kBK / 32; ks < kBK / 16; ++ks)
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + ks * 8, desc_mnmajor(va, ks), idesc(true), 1u);
        commit(&sm.o_done[t]);
      };
      wait_k(0);
      issue_s(0, 0);
      issue_s(1, 0);
      commit(&sm.k_empty[0]);
      for (int kb = 0; kb < nblk1; ++kb) {
        bar_wait(&sm.v_full[kb & 1], (kb >> 1) & 1);
        bool k_ready = false;
        if (kb < nblk0) {
          issue_pv(0, kb);
          if (kb + 1 < nblk0) {
            wait_k(kb + 1);
            k_ready = true;
            issue_s(0, kb + 1);
          }
        }
        issue_pv(1, kb);
        commit(&sm.v_empty[kb & 1]);
        if (kb + 1 < nblk1) {
          if (!k_ready) wait_k(kb + 1);
          issue_s(1, kb + 1);
          commit(&sm.k_empty[(kb + 1) & 1]);
        }
      }
    }
  } else if (warp >= 2 && warp < 10) {
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const int q0t = q0 + t * kBQ, qrow = q0t + r;
    const int nb = t ? nblk1 : nblk0;
    const uint32_t lb = (uint32_t)(quarter * 32) << 16;
    const uint32_t St = tmem + lb + t * 128, Ot = tmem + lb + 256 + t * 128;
    float m_run = -INFINITY, l_run = 0.0f;
    for (int kb = 0; kb < nb; ++kb) {
      bar_wait(&sm.s_full[t], kb & 1);
      fence_after();
      float sv[kBK];
      {
        uint32_t rr[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tld32(St + c * 32, rr[c]);
        tld_wait();
#pragma unroll
        for (int i = 0; i < kBK; ++i) sv[i] = __uint_as_float(rr[i >> 5][i & 31]);
      }
      if ((kb + 1) * kBK > q0t) {  // the diagonal block: keys past the row masked
        const int lim = qrow - kb * kBK;
#pragma unroll
        for (int i = 0; i < kBK; ++i)
          if (i > lim) sv[i] = -INFINITY;
      }
      float mp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mp[k] = -INFINITY;
#pragma unroll
      for (int i = 0; i < kBK; ++i) mp[i & 7] = fmaxf(mp[i & 7], sv[i]);
      const float mraw = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                               fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
      const float mx = fmaxf(m_run, mraw * scale_log2);
      const bool bump = mx > m_run + 8.0f;  // lazy rescaling, as in v2
      const float m_new = bump ? mx : m_run;
      const float corr = bump ? ex2(m_run - mx) : 1.0f;
      const float nm = -m_new;
      float ps[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int i = 64 * half; i < 64 * half + 64; ++i) {
          const float x = fmaf(sv[i], scale_log2, nm);
          sv[i] = ex2(x);
          ps[i & 7] += sv[i];
        }
        uint32_t pk[32];  // this half of P_t -> TMEM over S_t (32 columns of bf16 pairs)
#pragma unroll
        for (int k = 0; k < 32; ++k) pk[k] = pack(sv[64 * half + 2 * k], sv[64 * half + 2 * k + 1]);
        tst32(St + half * 32, pk);
        // O is rescaled before the first half of PV(kb) may accumulate into
        // it (after the first half's P is packed, so its registers are free)
        if (half == 0 && kb > 0 && __any_sync(0xffffffffu, bump)) {  // PV_t(kb-1) is complete (see above)
#pragma unroll
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t rr[32];
            tld32(Ot + c * 32, rr);
            tld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * corr);
            tst32(Ot + c * 32, rr);
          }
        }
        tst_wait();
        fence_before();
        bar_arrive(half ? &sm.p_hi[t] : &sm.p_lo[t]);
      }
      l_run = l_run * corr + (((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7])));
      m_run = m_new;
    }
    // After the last arrive o_done[t] is in phase nb-1 (PV_t(nb-1) pending)
    // or nb; earlier phases completed before S_t(nb-1) did.
    bar_wait(&sm.o_done[t], (nb - 1) & 1);
    fence_after();
    // O_t / l -> bf16 through shared memory (Q_t: every MMA reading it has
    // completed once o_done[t] has) and two TMA stores of full lines
    stage_rows_bf16(Ot, 1.0f / l_run, sm.Q[t], r);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) asm volatile("bar.sync 5, 128;" ::: "memory");  // this warpgroup only
    else asm volatile("bar.sync 6, 128;" ::: "memory");
    if (r == 0) store_tile_128(&map_o, sm.Q[t], j * kD, row0 + q0t);
    lse[(long long)bh * s + qrow] = (m_run + log2f(l_run)) * 0.6931471805599453f;
  }
  fence_before();
  __syncthreads();
  cta_stamp(tr, 2);
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ============================================================== backward
// One CTA per (128-key block, batch x head); loop over 64-query blocks from
// the diagonal down.  Per block (TMEM columns in brackets):
//   S^T  = K Q^T            [0,64)     dP^T = V dO^T          [64,128)
//   P^T  = exp(S^T*scale - lse_q), dS^T = P^T (dP^T - D_q)   (registers,
//          thread = key row; written bf16 to shared memory)
//   dV  += P^T dO           [128,256)  dK  += dS^T Q          [256,384)
//   dQ^T = K^T dS^T         [384,448)  -> fp32 red.add into dq_acc
// The dS^T bytes serve as the K-major A operand of dK and as the MN-major
// operand of dQ^T.  lse and D (= rowsum(dO*O)) of each query block arrive by
// bulk copy with the Q / dO tiles.
constexpr int kBQb = 64;                      // queries per backward block
constexpr int kHalf = kBQb * kD * 2;          // 16 KB: 64 x 128 bf16
constexpr int kPT = kBK * kBQb * 2;           // 16 KB: 128 keys x 64 queries bf16


__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
// K-major tile of 64-element K chunks, `rows` rows per chunk (chunk stride
// rows*128 B); k-step ks moves 32 B inside the swizzle row.
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int ks, int rows) {
  return sdesc(base + (ks >> 2) * rows * 128 + (ks & 3) * 32, 16, 1024);
}
// MN-major operand: 64-element MN blocks of [k-rows][128 B] (LBO = block
// stride), k-step of 16 rows.
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int ks, uint32_t lbo) {
  return sdesc(base + ks * 16 * 128, lbo, 1024);
}
constexpr uint32_t idesc2(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

constexpr int kThreadsBwd = 384;  // warps 0 TMA, 1 MMA, 2 TMEM alloc, 4-7 softmax, 8-11 dQ drain
// ---------------------------------------------------------- backward v3
// Same math; the MMA issue order and buffering are arranged so that neither
// the Q/dO loads nor the dQ drain sit on the tensor pipe's critical path:
//   per block i the MMA warp issues dQ^T(i) first (commit dq_full), then
//   dV(i), dK(i) (commit q_empty / pds_empty), then S^T/dP^T(i+2).  The drain
//   of dQ^T(i) overlaps dV/dK(i); the softmax of block i+1 overlaps
//   dQ/dV/dK(i); the single P^T/dS^T buffer is rewritten while S/dP(i+2)
//   run; Q/dO/L/D use a 3-slot ring so block i+2's loads start one block
//   earlier than in v2.  dQ^T leaves through a 32-query fp32 staging half.
//   TMEM: [0,128)/[128,256) S^T|dP^T of block i&1 (dQ^T(i) overwrites the
//   S^T half after the softmax read it), [256,384) dV, [384,512) dK.
// ---------------------------------------------------------- backward v4
// v3 with P^T kept in tensor memory: the softmax warps tcgen05.st P^T (bf16
// pairs) over the dP^T half they have just read, and dV += P^T dO runs as a
// TS-MMA (A operand from TMEM).  That frees the P^T shared-memory tile and,
// with a 16-query dQ staging tile, pays for a 4-slot Q / dO ring, so the
// ~2k-cycle TMA round trip of block i+4 overlaps two block periods.
// v3 description (unchanged parts):
// Same math; the MMA issue order and buffering are arranged so that neither
// the Q/dO loads nor the dQ drain sit on the tensor pipe's critical path:
//   per block i the MMA warp issues dQ^T(i) first (commit dq_full), then
//   dV(i), dK(i) (commit q_empty / pds_empty), then S^T/dP^T(i+2).  The drain
//   of dQ^T(i) overlaps dV/dK(i); the softmax of block i+1 overlaps
//   dQ/dV/dK(i); the single P^T/dS^T buffer is rewritten while S/dP(i+2)
//   run; Q/dO/L/D use a 3-slot ring so block i+2's loads start one block
//   earlier than in v2.  dQ^T leaves through a 32-query fp32 staging half.
//   TMEM: [0,128)/[128,256) S^T|dP^T of block i&1 (dQ^T(i) overwrites the
//   S^T half after the softmax read it), [256,384) dV, [384,512) dK.
constexpr int kQS4 = 4;  // Q / dO ring depth
constexpr int kDqRows4 = kBQb / 4;  // dQ staging rows
struct FaBwdSmem4 {
  uint8_t K[kTile], V[kTile];
  uint8_t Q[kQS4][kHalf], dO[kQS4][kHalf];
  uint8_t dST[kPT];
  float dq_stage[2][kDqRows4][kD];  // double-buffered: piece p+1 is written while piece p's reduce reads
  float L[kQS4][kBQb], D[kQS4][kBQb];
  uint64_t kv_full, q_full[kQS4], q_empty[kQS4], s_full[2], ps_full, pds_empty, dq_full[2], dq_empty[2], mma_done;
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreadsBwd, 1)
    fa_bwd_tc4_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_q,
                      const __grid_constant__ CUtensorMap map_do, const __grid_constant__ CUtensorMap map_dq,
                      const __grid_constant__ CUtensorMap map_out,
                      const float* __restrict__ lse, const float* __restrict__ Dg, bf16* __restrict__ dqkv, int s,
                      int h, int H, float scale, long long* __restrict__ tr) {
  pdl_trigger_and_wait();
  extern __shared__ __align__(1024) uint8_t rawb4[];
  FaBwdSmem4& sm = *reinterpret_cast<FaBwdSmem4*>(rawb4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.y;  // grid (b*H, s/128): key block 0 (most query blocks) first
  const int bh = blockIdx.x, bi = bh / H, j = bh % H;
  const int row0 = bi * s;
  const int k0 = kb * kBK;
  const int qb0 = k0 / kBQb, nq = s / kBQb - qb0;
  const float scale_log2 = scale * 1.4426950408889634f;
  // GS_ATTN_TRACE diagnostics: clock64 stamps of CTA (0, 0)'s pipeline events
  // tr[ev * 64 + i]: 0 mma ps_full(i) seen, 1 mma S(i) issued, 2 softmax
  // s_full(i) seen, 3 softmax math done, 4 softmax P/dS written, 5 drain
  // dq_full(i) seen, 6 drain dq_empty(i) arrived, 7 producer Q(i) issued
  cta_stamp(tr, 1);
  long long* trc = (tr && blockIdx.x == 0 && blockIdx.y == 0) ? tr : nullptr;
#define GS_TR4(ev, i)                                            \
  do {                                                           \
    if (trc && (i) < 64) trc[(ev) * 64 + (i)] = clock64();       \
  } while (0)

  if (threadIdx.x == 0) {
    bar_init(&sm.kv_full, 1);
    for (int i = 0; i < kQS4; ++i) {
      bar_init(&sm.q_full[i], 1);
      bar_init(&sm.q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(&sm.s_full[i], 1);
      bar_init(&sm.dq_full[i], 1);
      bar_init(&sm.dq_empty[i], 128);
    }
    bar_init(&sm.ps_full, 128);
    bar_init(&sm.pds_empty, 1);
    bar_init(&sm.mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Thread 0 is also the producer: it starts the K / V tiles and the first
  // ring slots before the CTA-wide sync, so their latency overlaps the TMEM
  // allocation (the first tiles of a CTA were ~1.3k cycles late otherwise).
  auto load_q = [&](int i) {
    const int sl = i % kQS4, q0 = (qb0 + i) * kBQb;
    bar_expect(&sm.q_full[sl], 2 * kHalf + 2 * kBQb * 4);
    for (int c = 0; c < 2; ++c) {
      tma2d(sm.Q[sl] + c * 8192, &map_q, &sm.q_full[sl], j * kD + 64 * c, row0 + q0);
      tma2d(sm.dO[sl] + c * 8192, &map_do, &sm.q_full[sl], j * kD + 64 * c, row0 + q0);
    }
    bulk_g2s(sm.L[sl], lse + (long long)bh * s + q0, kBQb * 4, &sm.q_full[sl]);
    bulk_g2s(sm.D[sl], Dg + (long long)bh * s + q0, kBQb * 4, &sm.q_full[sl]);
    GS_TR4(7, i);
  };
  const int n_early = nq < kQS4 ? nq : kQS4;  // ring slots that start empty
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_do)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    bar_expect(&sm.kv_full, 2 * kTile);
    for (int c = 0; c < 2; ++c) {
      tma2d(sm.K + c * 16384, &map_qkv, &sm.kv_full, h + j * kD + 64 * c, row0 + k0);
      tma2d(sm.V + c * 16384, &map_qkv, &sm.kv_full, 2 * h + j * kD + 64 * c, row0 + k0);
    }
    for (int i = 0; i < n_early; ++i) load_q(i);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem;
  constexpr uint32_t kDV = 256, kDK = 384;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = n_early; i < nq; ++i) {
        bar_wait(&sm.q_empty[i % kQS4], ((i / kQS4) & 1) ^ 1);
        load_q(i);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t ka = su32(sm.K), va = su32(sm.V), da = su32(sm.dST);
      bar_wait(&sm.kv_full, 0);
      auto issue_s = [&](int i) {  // S^T, dP^T of block i into TMEM buffer i&1
        const int buf = i & 1, sl = i % kQS4;
        bar_wait(&sm.q_full[sl], (i / kQS4) & 1);
        bar_wait(&sm.dq_empty[buf], ((i >> 1) & 1) ^ 1);  // dQ^T of block i-2 drained
        GS_TR4(1, i);
        fence_after();
        const uint32_t qa = su32(sm.Q[sl]), oa = su32(sm.dO[sl]);
        const uint32_t t0 = tmem + buf * 128;
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks) {
          mma(t0, desc_k(ka, ks, 128), desc_k(qa, ks, 64), idesc2(64, false, false), ks != 0);
          mma(t0 + 64, desc_k(va, ks, 128), desc_k(oa, ks, 64), idesc2(64, false, false), ks != 0);
        }
        commit(&sm.s_full[buf]);
      };
      issue_s(0);
      if (nq > 1) issue_s(1);
      for (int i = 0; i < nq; ++i) {
        const int buf = i & 1, sl = i % kQS4;
        bar_wait(&sm.ps_full, i & 1);
        GS_TR4(0, i);
        fence_after();
        // dQ^T(i) = K^T dS^T into the (already read) S^T half of buffer i&1
#pragma unroll
        for (int ks = 0; ks < kBK / 16; ++ks)
          mma(tmem + buf * 128, desc_mn(ka, ks, 16384), desc_mn(da, ks, 8192), idesc2(64, true, true), ks != 0);
        commit(&sm.dq_full[buf]);
        const uint32_t qa = su32(sm.Q[sl]), oa = su32(sm.dO[sl]);
#pragma unroll
        for (int ks = 0; ks < kBQb / 16; ++ks) {
          // A = P^T in TMEM (dP^T half of buffer i&1, 8 columns per 16 queries)
          mma_ts(tmem + kDV, tmem + buf * 128 + 64 + ks * 8, desc_mn(oa, ks, 8192), idesc2(128, false, true),
                 (i | ks) != 0);
          mma(tmem + kDK, desc_k(da, ks, 128), desc_mn(qa, ks, 8192), idesc2(128, false, true), (i | ks) != 0);
        }
        commit(&sm.q_empty[sl]);
        commit(&sm.pds_empty);
        if (i + 2 < nq) issue_s(i + 2);
      }
      commit(&sm.mma_done);
    }
  } else if (warp >= 4 && warp < 8) {
    const int r = (warp - 4) * 32 + lane;  // key row
    const uint32_t lb = ((uint32_t)((warp & 3) * 32)) << 16;
    const int key = k0 + r;
    const uint32_t swz = (uint32_t)(r & 7);
    const int rowoff = (r >> 3) * 1024 + (r & 7) * 128;
    for (int i = 0; i < nq; ++i) {
      const int buf = i & 1, sl = i % kQS4, q0 = (qb0 + i) * kBQb;
      bar_wait(&sm.q_full[sl], (i / kQS4) & 1);  // L, D of this block
      bar_wait(&sm.s_full[buf], (i >> 1) & 1);
      if (r == 0) GS_TR4(2, i);
      fence_after();
      float p[kBQb], ds[kBQb];
      // only the two query blocks on the diagonal (i < 2) hold masked pairs
      const bool diag = q0 < k0 + kBK;
#pragma unroll
      for (int c = 0; c < kBQb / 32; ++c) {
        uint32_t a[32], b[32];
        tld32(tmem + lb + buf * 128 + c * 32, a);
        tld32(tmem + lb + buf * 128 + 64 + c * 32, b);
        tld_wait();
        if (diag) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int qi = c * 32 + q;
            float pv = ex2(fmaf(__uint_as_float(a[q]), scale_log2, -sm.L[sl][qi]));
            if (q0 + qi < key) pv = 0.0f;  // causal
            p[qi] = pv;
            ds[qi] = pv * (__uint_as_float(b[q]) - sm.D[sl][qi]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int qi = c * 32 + q;
            const float pv = ex2(fmaf(__uint_as_float(a[q]), scale_log2, -sm.L[sl][qi]));
            p[qi] = pv;
            ds[qi] = pv * (__uint_as_float(b[q]) - sm.D[sl][qi]);
          }
        }
      }
      if (r == 0) GS_TR4(3, i);
      {  // P^T -> TMEM over the consumed dP^T half (lane = key row)
        uint32_t pk[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) pk[k] = pack(p[2 * k], p[2 * k + 1]);
        tst32(tmem + lb + buf * 128 + 64, pk);
      }
      bar_wait(&sm.pds_empty, (i & 1) ^ 1);  // MMAs of block i-1 done with dS^T
#pragma unroll
      for (int pc = 0; pc < 8; ++pc) {
        const float* w = ds + pc * 8;
        *reinterpret_cast<uint4*>(sm.dST + rowoff + ((pc ^ swz) << 4)) =
            make_uint4(pack(w[0], w[1]), pack(w[2], w[3]), pack(w[4], w[5]), pack(w[6], w[7]));
      }
      tst_wait();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      fence_before();
      bar_arrive(&sm.ps_full);
      if (r == 0) GS_TR4(4, i);
    }
    bar_wait(&sm.mma_done, 0);
    fence_after();
    // dK leaves through shared memory and two TMA stores (full 128-B lines):
    // per-thread row stores of 16 B into 12 KB-strided rows took ~4.5k
    // cycles.  The Q ring is free once every MMA has completed.
    stage_rows_bf16(tmem + lb + kDK, scale, sm.Q[0], r);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 4, 128;" ::: "memory");
    if (r == 0) store_tile_128(&map_out, sm.Q[0], h + j * kD, row0 + k0);
  } else if (warp >= 8) {
    const int r = (warp - 8) * 32 + lane;  // d row of dQ^T; key row for dV
    const uint32_t lb = ((uint32_t)((warp & 3) * 32)) << 16;
    for (int i = 0; i < nq; ++i) {
      const int buf = i & 1;
      bar_wait(&sm.dq_full[buf], (i >> 1) & 1);
      if (r == 0) GS_TR4(5, i);
      fence_after();
      uint32_t rr[kBQb];
      tld32(tmem + lb + buf * 128, *reinterpret_cast<uint32_t(*)[32]>(rr));
      tld32(tmem + lb + buf * 128 + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
      tld_wait();
      fence_before();
      bar_arrive(&sm.dq_empty[buf]);  // TMEM buffer free for S/dP(i+2)
      if (r == 0) GS_TR4(6, i);
#pragma unroll
      for (int half = 0; half < kBQb / kDqRows4; ++half) {
        const int sb = half & 1;  // pieces per block is even: piece parity == half parity
        // the reduce that last read this buffer (two pieces back) is done
        if (r == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 3, 128;" ::: "memory");
#pragma unroll
        for (int q = 0; q < kDqRows4; ++q) sm.dq_stage[sb][q][r] = __uint_as_float(rr[half * kDqRows4 + q]) * scale;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 3, 128;" ::: "memory");
        if (r == 0) {
          const int q0 = (qb0 + i) * kBQb + half * kDqRows4;
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&map_dq)),
              "r"(su32(&sm.dq_stage[sb][0][0])), "r"(j * kD), "r"(row0 + q0)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (r == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    bar_wait(&sm.mma_done, 0);
    fence_after();
    stage_rows_bf16(tmem + lb + kDV, 1.0f, sm.dO[0], r);  // dV, same path as dK (dO ring)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 3, 128;" ::: "memory");
    if (r == 0) store_tile_128(&map_out, sm.dO[0], 2 * h + j * kD, row0 + k0);
  }
  fence_before();
  __syncthreads();
  cta_stamp(tr, 2);
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

}  // namespace

// The tcgen05 path: bf16, head_dim 128, s a multiple of the forward's two
// 128-query tiles (every BASELINE geometry); anything else runs the generic
// SIMT kernels (attention.cu), which also serve the fp32 parity mode.
bool attention_tc_supported(DType dt, int s, int h, int H) {
  return dt == DType::BF16 && h % H == 0 && h / H == kD && s % (2 * kBQ) == 0 && encoder() != nullptr;
}


// GS_ATTN_TRACE=1: clock64 timeline of CTA (0,0) of the backward (stderr)
// Past the 8 x 64 event stamps, every CTA writes {smid, start, end}
// (%globaltimer ns) at tr[512 + 4 * cta]: the whole-grid schedule.
static long long* attn_trace_begin(cudaStream_t st, int ncta) {
  static const bool on = getenv("GS_ATTN_TRACE") != nullptr;
  if (!on) return nullptr;
  long long* tr = nullptr;
  const size_t n = 8 * 64 + 4 * (size_t)ncta;
  cudaMalloc(&tr, n * sizeof(long long));
  cudaMemsetAsync(tr, 0, n * sizeof(long long), st);
  return tr;
}
static void attn_trace_end(long long* tr, cudaStream_t st, int ncta, int ny,
                           const char* legend = "0 mma_ps_full 1 mma_S_issue 2 sm_s_full 3 sm_math 4 sm_written "
                                                "5 dq_full 6 dq_empty 7 prod_Q",
                           int t0_event = 7) {
  if (!tr) return;
  long long hbuf[8 * 64];
  std::vector<long long> cta(4 * (size_t)ncta);
  cudaMemcpyAsync(hbuf, tr, sizeof(hbuf), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(cta.data(), tr + 8 * 64, cta.size() * sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(tr);
  {  // grid schedule: span, SM occupancy, CTA durations per blockIdx.y
    long long t_lo = LLONG_MAX, t_hi = 0, last_start = 0, busy = 0;
    std::vector<double> dur_y(ny, 0.0);
    std::vector<int> n_y(ny, 0);
    for (int c = 0; c < ncta; ++c) {
      const long long a = cta[4 * c + 1], e = cta[4 * c + 2];
      t_lo = std::min(t_lo, a);
      t_hi = std::max(t_hi, e);
      last_start = std::max(last_start, a);
      busy += e - a;
      dur_y[c / (ncta / ny)] += (double)(e - a);
      n_y[c / (ncta / ny)] += 1;
    }
    fprintf(stderr, "[attn grid] ctas %d span %.1f us, last CTA starts at %.1f us, sum CTA time / (span x 148 SMs) = %.2f CTAs per SM\n",
            ncta, (t_hi - t_lo) / 1e3, (last_start - t_lo) / 1e3, (double)busy / ((double)(t_hi - t_lo) * 148));
    for (int y = 0; y < ny; ++y)
      fprintf(stderr, "[attn grid] blockIdx.y %2d: mean CTA %.1f us\n", y, n_y[y] ? dur_y[y] / n_y[y] / 1e3 : 0.0);
  }
  const long long t0 = hbuf[t0_event * 64];
  fprintf(stderr, "[attn trace] ev: %s\n", legend);
  for (int i = 0; i < 32; ++i) {
    fprintf(stderr, "[attn trace] %2d", i);
    for (int ev = 0; ev < 8; ++ev) fprintf(stderr, " %7lld", hbuf[ev * 64 + i] ? hbuf[ev * 64 + i] - t0 : -1);
    fprintf(stderr, "\n");
  }
}

cudaError_t attention_fwd_tc(const void* qkv, void* o, float* lse, int b, int s, int h, int H, cudaStream_t st) {
  if (!attention_tc_supported(DType::BF16, s, h, H)) return cudaErrorInvalidValue;
  CUtensorMap mq;  // Q / K / V columns of qkv, 64-column x 128-row boxes
  const cuuint64_t dims[2] = {(cuuint64_t)3 * h, (cuuint64_t)b * s};
  const cuuint64_t strides[1] = {(cuuint64_t)3 * h * 2};
  const cuuint32_t elem[2] = {1, 1};
  {
    const cuuint32_t box[2] = {64, 128};
    if (encoder()(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int smem3 = (int)sizeof(FaSmem3);
  static bool init3 = false;
  if (!init3) {
    cudaError_t e = cudaFuncSetAttribute(fa_fwd_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    if (e != cudaSuccess) return e;
    init3 = true;
  }
  count_launch();
  const int ny = s / (2 * kBQ);
  long long* tr = attn_trace_begin(st, b * H * ny);
  CUtensorMap mo;  // o, bf16, 64-column x 128-row boxes (TMA stores of O)
  {
    const cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)b * s};
    const cuuint64_t strides[1] = {(cuuint64_t)h * 2};
    const cuuint32_t box[2] = {64, 128};
    if (encoder()(&mo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, o, dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  cudaError_t le = launch_pdl(fa_fwd_tc3_kernel, dim3(b * H, ny), dim3(kThreadsF3), smem3, st, mq, mo, (bf16*)o, lse,
                              s, h, H, 1.4426950408889634f / sqrtf((float)kD), tr);
  if (le != cudaSuccess) return le;
  attn_trace_end(tr, st, b * H * ny, ny, "(v3: grid schedule only)", 0);
  return cudaGetLastError();
}

// dqkv: writes the dK / dV columns; dq_acc (fp32 [b*s][h], zeroed by the
// caller) receives dQ; D = rowsum(dO * O) per (bh, q).
cudaError_t attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* lse2, const float* D,
                             void* dqkv,
                             float* dq_acc, int b, int s, int h, int H, cudaStream_t st) {
  CUtensorMap mq, mq64, md;
  const cuuint32_t elem[2] = {1, 1};
  for (int rows : {128, 64}) {
    const cuuint64_t dims[2] = {(cuuint64_t)3 * h, (cuuint64_t)b * s};
    const cuuint64_t strides[1] = {(cuuint64_t)3 * h * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)rows};
    if (encoder()(rows == 128 ? &mq : &mq64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims,
                  strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)b * s};
    const cuuint64_t strides[1] = {(cuuint64_t)h * 2};
    const cuuint32_t box[2] = {64, 64};
    if (encoder()(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dout), dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  CUtensorMap mdq;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)b * s};
    const cuuint64_t strides[1] = {(cuuint64_t)h * 4};
    const cuuint32_t box[2] = {128, (cuuint32_t)kDqRows4};
    if (encoder()(&mdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const int smem4 = (int)sizeof(FaBwdSmem4);
    static bool init4 = false;
    if (!init4) {
      cudaError_t e = cudaFuncSetAttribute(fa_bwd_tc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
      if (e != cudaSuccess) return e;
      init4 = true;
    }
    count_launch();
    long long* tr = attn_trace_begin(st, b * H * (s / kBK));
    CUtensorMap mout;  // dqkv, bf16, 64-column x 128-row boxes (dK / dV TMA stores)
    {
      const cuuint64_t dims[2] = {(cuuint64_t)3 * h, (cuuint64_t)b * s};
      const cuuint64_t strides[1] = {(cuuint64_t)3 * h * 2};
      const cuuint32_t box[2] = {64, 128};
      if (encoder()(&mout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dqkv, dims, strides, box, elem,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    cudaError_t le = launch_pdl(fa_bwd_tc4_kernel, dim3(b * H, s / kBK), dim3(kThreadsBwd), smem4, st, mq, mq64, md,
                                mdq, mout, lse2, D, (bf16*)dqkv, s, h, H, 1.0f / sqrtf((float)kD), tr);
    if (le != cudaSuccess) return le;
    attn_trace_end(tr, st, b * H * (s / kBK), s / kBK);
    return cudaGetLastError();
  }
}

}  // namespace gs
