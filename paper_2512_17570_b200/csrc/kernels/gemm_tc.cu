// sm_100a tensor-core GEMM for the bf16 layer executor:
//   TMA (cp.async.bulk.tensor, 128B swizzle) -> 4-stage shared-memory ring
//   -> tcgen05.mma.cta_group::1.kind::f16 issued by one elected thread
//   -> fp32 accumulators in TMEM (two buffers, so the epilogue of tile i
//      overlaps the MMAs of tile i+1) -> tcgen05.ld epilogue warps with the
//      layer's fused epilogues (residual add, GELU, fp32 gradient accumulate).
// Persistent: one CTA per SM walks the output tiles.  Operands may be
// K-major or MN-major (transposed) so forward (X W^T), data-gradient (dY W)
// and weight-gradient (dY^T X) all run without transpose copies.
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace gs {

namespace {

using bf16 = __nv_bfloat16;

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, one per column half
constexpr int kEpiWarpsCfg = kEpiWarps;
constexpr int kThreads = 128 + 32 * kEpiWarps;

// CG = 1: one CTA computes a 128 x BN tile.  CG = 2: a CTA pair (cluster of
// 2, tcgen05 cta_group::2) computes 256 x BN; each SM stages 128 rows of A and
// BN/2 rows of B, the MMA exchanges B halves between the pair.
template <int BN, int CG = 1> struct TileCfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = (BN / CG) * BK * 2;
  static constexpr int kStages = (kABytes + kBBytes) <= 32768 ? 6 : 4;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // double-buffered accumulator; allocations are powers of two >= 32 columns
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  // epilogue staging for TMA stores: 4 KB per epilogue warp (32 rows x 128 B)
  static constexpr int kEpiStage = 4096;
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiWarpsCfg * kEpiStage + 1024 /*align*/ + 256 /*barriers*/;
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 2-SM form: executed by both CTAs of the pair; bytes land in the issuing
// CTA's smem and complete on CTA 0's barrier (peer bit 24 cleared).
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread i gets its lane's 32 values.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Operand tile in shared memory, as the UMMA reads it for k-step `ks`
// (16 elements of K):
//  K-major : rows of 128 B (64 K-elements), 8-row atoms of 1 KB; the k-step
//            moves the start address 32 B inside the swizzle atom.
//  MN-major: 64-element MN blocks, each [BK rows][128 B]; 8 K-rows per atom;
//            LBO = distance between MN blocks, SBO = between 8-row K groups.
template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int ks) {
  if (!MN) return smem_desc(base + ks * 32, 16, 1024);
  return smem_desc(base + ks * 16 * 128, BK * 128, 1024);
}

template <int BN, bool A_MN, bool B_MN, int CG = 1>
__host__ __device__ constexpr uint32_t instr_desc() {
  return (1u << 4)            // D format f32
         | (1u << 7)          // A bf16
         | (1u << 10)         // B bf16
         | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)((BM * CG) >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Work list of one persistent unit (a CTA, or a CTA pair for CG = 2).
// Tiles [0, dp) are data-parallel (whole tiles, round-robin over units).  The
// last `rem` tiles are stream-K: their rem * kt k-blocks are cut into `units`
// contiguous, equal ranges, so the tail wave is spread over every SM instead
// of leaving (1 - rem / units) of them idle.  A range covers at most two
// tiles (rem < units); the unit whose range holds a tile's last k-block owns
// the tile: it adds the fp32 partials of the earlier pieces (workspace slot =
// the writer's CTA, readiness flag = launch epoch) before the fused epilogue.
// Every unit has at most one non-owner piece, always its last item, and an
// owner only waits on lower units, so the waits form no cycle.
struct Sched {
  int unit, units, kt, rem, dp;
  __device__ __forceinline__ int n_dp() const { return unit < dp ? (dp - 1 - unit) / units + 1 : 0; }
  __device__ __forceinline__ long long sk_bound(int u) const { return (long long)u * rem * kt / units; }
  // item i of this unit: tile t, k-blocks [ka, kb)
  __device__ __forceinline__ bool item(int i, int& t, int& ka, int& kb) const {
    const int nd = n_dp();
    if (i < nd) {
      t = unit + i * units;
      ka = 0;
      kb = kt;
      return true;
    }
    if (rem == 0) return false;
    const long long l1 = sk_bound(unit + 1);
    long long l = sk_bound(unit);
    for (int j = nd; l < l1; ++j) {
      const int ts = (int)(l / kt), a = (int)(l % kt);
      const int b = (int)((long long)a + (l1 - l) < kt ? (long long)a + (l1 - l) : kt);
      if (j == i) {
        t = dp + ts;
        ka = a;
        kb = b;
        return true;
      }
      l += b - a;
    }
    return false;
  }
};

// Output tile t -> (m tile, n tile), grouped raster: runs of kGroupM m-tiles
// sweep the n columns, so one wave of ~74-148 units touches ~8 A row panels
// and ~10 B column panels — an L2-sized working set even when K is large
// (8192^3: the m-fastest raster streamed ~300 MB of A panels per wave).
constexpr int kGroupM = 8;
__device__ __forceinline__ void tile_coords(int t, int mt, int nt, int& tm, int& tn) {
  const int per_group = kGroupM * nt;
  const int g = t / per_group, first = g * kGroupM;
  const int rows = min(mt - first, kGroupM);
  const int r = t - g * per_group;
  tm = first + r % rows;
  tn = r / rows;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Epilogue of one 32-row x 32-column accumulator chunk of an epilogue warp
// (thread = row, v = its 32 fp32 columns): fused math in registers, then the
// warp stages the chunk in shared memory (TMA swizzle layout: 64 B rows with
// SWIZZLE_64B for bf16, 128 B rows with SWIZZLE_128B for fp32, which makes
// the row-per-thread 16-byte stores bank-conflict free) and lane 0 issues a
// TMA store (fp32 accumulate: a TMA reduce-add, no read-back) of full lines.
template <int EPI>
__device__ __forceinline__ void epilogue_store(const float (&v)[32], int lane, int row, int col, int row0, int M, int ldc,
                                               const bf16* R, uint8_t* stg, const CUtensorMap* map_c,
                                               const CUtensorMap* map_g) {
  const uint32_t sa = smem_u32(stg);
  // the previous chunk's bulk store must have finished reading the staging
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
  if constexpr (EPI == (int)Epi::AccumF32 || EPI == (int)Epi::StoreF32) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t a = sa + lane * 128 + ((j ^ (lane & 7)) << 4);
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v[4 * j]), "f"(v[4 * j + 1]),
                   "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                   : "memory");
    }
  } else {
    float w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = v[i];
    if constexpr (EPI == (int)Epi::AddResidual || EPI == (int)Epi::MulGeluGrad) {
      // rows past M (half-empty last pair tile) read row 0; the store clips them
      const uint4* r = reinterpret_cast<const uint4*>(R + (long long)(row < M ? row : 0) * ldc + col);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 x = r[q];
        const uint32_t u[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162*>(&u[k]);
          if (EPI == (int)Epi::AddResidual) {
            w[8 * q + 2 * k] += __bfloat162float(p.x);
            w[8 * q + 2 * k + 1] += __bfloat162float(p.y);
          } else {
            // round dg to bf16 first: identical to storing dg and running gelu_bwd
            w[8 * q + 2 * k] = __bfloat162float(__float2bfloat16_rn(w[8 * q + 2 * k])) * gelu_grad_fast(__bfloat162float(p.x));
            w[8 * q + 2 * k + 1] =
                __bfloat162float(__float2bfloat16_rn(w[8 * q + 2 * k + 1])) * gelu_grad_fast(__bfloat162float(p.y));
          }
        }
      }
    }
    if constexpr (EPI == (int)Epi::Gelu) {  // the G of StoreGelu, without storing u
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = gelu_fast(__bfloat162float(__float2bfloat16_rn(w[i])));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t a = sa + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack_bf16(w[8 * j], w[8 * j + 1])),
                   "r"(pack_bf16(w[8 * j + 2], w[8 * j + 3])), "r"(pack_bf16(w[8 * j + 4], w[8 * j + 5])),
                   "r"(pack_bf16(w[8 * j + 6], w[8 * j + 7]))
                   : "memory");
    }
    if constexpr (EPI == (int)Epi::StoreGelu) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = gelu_fast(__bfloat162float(__float2bfloat16_rn(w[8 * j + k])));
        const uint32_t a = sa + 2048 + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack_bf16(r[0], r[1])),
                     "r"(pack_bf16(r[2], r[3])), "r"(pack_bf16(r[4], r[5])), "r"(pack_bf16(r[6], r[7]))
                     : "memory");
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
  __syncwarp();
  if (lane == 0) {
    if constexpr (EPI == (int)Epi::AccumF32)
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(map_c)),
                   "r"(sa), "r"(col), "r"(row0)
                   : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(map_c)),
                   "r"(sa), "r"(col), "r"(row0)
                   : "memory");
    if constexpr (EPI == (int)Epi::StoreGelu)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(map_g)),
                   "r"(sa + 2048), "r"(col), "r"(row0)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_g, int M,
                   int N, int K, void* C, const bf16* R, bf16* G, int ldc, int sk_rem, float4* __restrict__ sk_ws,
                   int* __restrict__ sk_flags, int sk_epoch, unsigned long long* span) {
  pdl_trigger_and_wait();
  if (span && threadIdx.x == 0) atomicMin(span, globaltimer_ns());
  using Cfg = TileCfg<BN, CG>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint8_t* smem_epi = smem + S * Cfg::kStageBytes;  // 1024-aligned: stage bytes are multiples of 1 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * Cfg::kEpiStage);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // M % 128 == 0; a CTA pair's last M tile may be half outside M (TMA loads
  // fill zeros, TMA stores clip, residual loads are guarded)
  const int mt = (M + BM * CG - 1) / (BM * CG), nt = N / BN, kt = K / BK;
  const int tiles = mt * nt;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;  // CTA within the pair
  const int unit = CG == 2 ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int units = CG == 2 ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
  constexpr int kBN_local = BN / CG;  // B rows staged by this CTA
  const Sched sch{unit, units, kt, sk_rem, tiles - sk_rem};

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEpiWarps * CG);  // epilogue threads of both CTAs release the accumulator
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
        if constexpr (CG == 2) tma_load_2d_2sm(dst, map, bar, c0, c1);
        else tma_load_2d(dst, map, bar, c0, c1);
      };
      int t, ka, kb_end;
      for (int it = 0; sch.item(it, t, ka, kb_end); ++it) {
        int tm, tn;
        tile_coords(t, mt, nt, tm, tn);
        const int m0 = tm * BM * CG + static_cast<int>(rank) * BM;
        const int n0 = tn * BN + static_cast<int>(rank) * kBN_local;
        for (int kb = ka; kb < kb_end; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          // CTA 0's barrier collects the bytes of both CTAs of a pair
          if (rank == 0) mbar_expect_tx(&full[stage], Cfg::kStageBytes * CG);
          uint8_t* sa = smem_a + stage * Cfg::kABytes;
          uint8_t* sb = smem_b + stage * Cfg::kBBytes;
          const int k0 = kb * BK;
          if (!A_MN) {
            load(sa, &map_a, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) load(sa + j * BK * 128, &map_a, &full[stage], m0 + 64 * j, k0);
          }
          if (!B_MN) {
            load(sb, &map_b, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < kBN_local / 64; ++j) load(sb + j * BK * 128, &map_b, &full[stage], n0 + 64 * j, k0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ===== MMA issuer (one thread; CTA 0 of a pair issues for both SMs)
    constexpr uint32_t idesc = instr_desc<BN, A_MN, B_MN, CG>();
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int t, ka, kb_end;
    for (int it = 0; sch.item(it, t, ka, kb_end); ++it) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = ka; kb < kb_end; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem_a + stage * Cfg::kABytes);
          const uint32_t b0 = smem_u32(smem_b + stage * Cfg::kBBytes);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            if constexpr (CG == 2)
              tc_mma_pair(d_tmem, operand_desc<A_MN>(a0, ks), operand_desc<B_MN>(b0, ks), idesc,
                          (kb > ka || ks != 0) ? 1u : 0u);
            else
              tc_mma(d_tmem, operand_desc<A_MN>(a0, ks), operand_desc<B_MN>(b0, ks), idesc,
                     (kb > ka || ks != 0) ? 1u : 0u);
          }
          // frees the smem slot (of both CTAs) when these MMAs retire
          if constexpr (CG == 2) tc_commit_pair(&empty[stage]); else tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {  // accumulator ready for the epilogue(s)
        if constexpr (CG == 2) tc_commit_pair(&tfull[acc]); else tc_commit(&tfull[acc]);
      }
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ===== epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (= tile rows);
    // warps 4-7 take the first half of the columns, warps 8-11 the second
    const int q = warp & 3;
    const int c_begin = ((warp - 4) / 4) * (BN / 2);
    int acc = 0;
    uint32_t acc_phase = 0;
    const int ep = threadIdx.x - 128;  // 0..255
    const int my_cta = unit * CG + static_cast<int>(rank);
    uint8_t* stg = smem_epi + (warp - 4) * Cfg::kEpiStage;
    int t, ka, kb_end;
    int n_items = 0;
    while (sch.item(n_items, t, ka, kb_end)) ++n_items;
    // A unit's last item may be its non-owner stream-K piece, right after an
    // owner piece that waits on the next-lower unit's non-owner piece.  Drain
    // the non-owner piece first (it sits in the other TMEM buffer) so every
    // partial is published without waiting: otherwise the waits chain through
    // all units and serialise their epilogues.
    bool swap_last = false;
    if (n_items >= 2) {
      sch.item(n_items - 1, t, ka, kb_end);
      swap_last = kb_end < kt;
    }
    for (int k = 0; k < n_items; ++k) {
      const int it = (swap_last && k >= n_items - 2) ? (2 * n_items - 3 - k) : k;
      sch.item(it, t, ka, kb_end);
      acc = it & 1;
      acc_phase = static_cast<uint32_t>((it >> 1) & 1);
      int tm, tn;
      tile_coords(t, mt, nt, tm, tn);
      const int m0 = tm * BM * CG + static_cast<int>(rank) * BM, n0 = tn * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      // workspace float4 index of (warp, chunk, q4, lane): coalesced per warp
      auto ws_at = [&](int cta, int ci, int q4) {
        return sk_ws + (((size_t)cta * kEpiWarps + (warp - 4)) * (BN / 64) + ci) * 256 + q4 * 32 + lane;
      };
      if (kb_end < kt) {
        // non-owner stream-K piece: park the fp32 partial, publish it
#pragma unroll 1
        for (int c = c_begin, ci = 0; c < c_begin + BN / 2; c += 32, ++ci) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            __stcg(ws_at(my_cta, ci, q4), make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]));
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (ep == 0) st_release(sk_flags + my_cta, sk_epoch);
      } else {
        int first_c = unit, n_c = 0;  // contributing units [first_c, unit)
        if (ka > 0) {
          const long long S = (long long)(t - sch.dp) * kt;
          while (first_c > 0 && sch.sk_bound(first_c) > S) --first_c;
          n_c = unit - first_c;
          if (ep < n_c) {
            const int* f = sk_flags + (first_c + ep) * CG + static_cast<int>(rank);
            while (ld_acquire(f) != sk_epoch) {
            }
          }
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        }
#pragma unroll 1
        for (int c = c_begin, ci = 0; c < c_begin + BN / 2; c += 32, ++ci) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
          for (int u = 0; u < n_c; ++u) {  // fixed order: deterministic sums
            const int cta = (first_c + u) * CG + static_cast<int>(rank);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
              const float4 p = __ldcg(ws_at(cta, ci, q4));
              v[4 * q4] += p.x;
              v[4 * q4 + 1] += p.y;
              v[4 * q4 + 2] += p.z;
              v[4 * q4 + 3] += p.w;
            }
          }
          epilogue_store<EPI>(v, lane, row, n0 + c, m0 + q * 32, M, ldc, R, stg, &map_c, &map_g);
        }
      }
      tc_fence_before();
      if constexpr (CG == 2) mbar_arrive_cluster(&tempty[acc], 0); else mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // staged stores done
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::kTmemCols));
  }
  if (span && threadIdx.x == 0) atomicMax(span + 1, globaltimer_ns());
}

// ------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor [outer][inner] (inner contiguous), box {64, box_outer}.
bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {64, box_outer};
  const cuuint32_t elem[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, elem,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Stream-K workspace of one stream: a 128 x BN fp32 partial slot and a
// readiness flag per CTA; flags carry the launch epoch, so they never need
// resetting.  One per stream, because launches on one stream are ordered.
struct SkSlot {
  float4* ws = nullptr;
  int* flags = nullptr;
  int epoch = 0;
};
SkSlot* sk_slot(cudaStream_t s) {
  static std::mutex mu;
  static std::vector<std::pair<cudaStream_t, SkSlot*>> slots;
  std::lock_guard<std::mutex> g(mu);
  for (auto& p : slots)
    if (p.first == s) return p.second;
  SkSlot* k = new SkSlot;  // lives for the process (device buffers freed at exit)
  const size_t ws_bytes = (size_t)num_sms() * BM * 256 * sizeof(float);
  if (cudaMalloc(&k->ws, ws_bytes) != cudaSuccess || cudaMalloc(&k->flags, num_sms() * sizeof(int)) != cudaSuccess ||
      cudaMemset(k->flags, 0, num_sms() * sizeof(int)) != cudaSuccess) {
    delete k;
    return nullptr;
  }
  slots.emplace_back(s, k);
  return k;
}

// Number of stream-K tiles for `tiles` output tiles on `units` persistent
// units with kt k-blocks each.  Only launches that would leave more than
// half of the units idle (fewer tiles than units / 2: small-M or small-N
// GEMMs with long K) are split: for a multi-wave launch's partial tail the
// partial-tile traffic and owner fix-up cost more than the recovered wave
// (measured 7-12% slower at the GPT-1.3B shapes).  Every unit gets >= 4
// k-blocks.
int sk_tiles(int tiles, int units, int kt) {
  if (units <= 1 || 2 * tiles >= units) return 0;
  if ((long long)tiles * kt < 4LL * units) return 0;
  return tiles;
}

// Output tensor [M][ldc] (N columns used) for the epilogue's 32 x 32 TMA
// stores: bf16 with 64-byte rows (SWIZZLE_64B) or fp32 with 128-byte rows
// (SWIZZLE_128B), matching epilogue_store's staging layout.
bool make_out_map(CUtensorMap* map, const void* base, bool f32, uint64_t N, uint64_t M, uint64_t ldc) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {N, M};
  const cuuint64_t strides[1] = {ldc * (f32 ? 4 : 2)};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t elem[2] = {1, 1};
  return fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
            dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
            f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
cudaError_t launch(const GemmArgs& g, cudaStream_t s) {
  using Cfg = TileCfg<BN, CG>;
  constexpr int kBNl = BN / CG;
  CUtensorMap ma, mb, mc, mg;
  const bool ok_a = A_MN ? make_map(&ma, g.A, g.M, g.K, BK) : make_map(&ma, g.A, g.K, g.M, BM);
  const bool ok_b = B_MN ? make_map(&mb, g.B, g.N, g.K, BK) : make_map(&mb, g.B, g.K, g.N, kBNl);
  if (!ok_a || !ok_b) return cudaErrorInvalidValue;
  constexpr bool kF32 = EPI == (int)Epi::AccumF32 || EPI == (int)Epi::StoreF32;
  const uint64_t ldc = g.ldc ? g.ldc : g.N;
  if (!make_out_map(&mc, g.C, kF32, g.N, g.M, ldc)) return cudaErrorInvalidValue;
  mg = mc;
  if (EPI == (int)Epi::StoreGelu && !make_out_map(&mg, g.G, false, g.N, g.M, ldc)) return cudaErrorInvalidValue;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, EPI, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (CG == 2) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  const int tiles = ((g.M + BM * CG - 1) / (BM * CG)) * (g.N / BN);
  const int full_grid = num_sms() / CG * CG;
  int rem = sk_tiles(tiles, full_grid / CG, g.K / BK);
  SkSlot* sk = rem ? sk_slot(s) : nullptr;
  if (!sk) rem = 0;
  int grid = rem ? full_grid : (tiles * CG < num_sms() ? tiles * CG : num_sms());
  grid = grid / CG * CG;
  int epoch = 0;
  if (sk) {
    if (++sk->epoch <= 0) sk->epoch = 1;
    epoch = sk->epoch;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl_trigger_and_wait
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mg, g.M, g.N, g.K, g.C, (const bf16*)g.R, (bf16*)g.G,
                            g.ldc ? g.ldc : g.N, rem, sk ? sk->ws : nullptr, sk ? sk->flags : nullptr, epoch, g.span);
}

template <int BN, bool A_MN, bool B_MN, int CG>
cudaError_t launch_epi(const GemmArgs& g, cudaStream_t s) {
  switch (g.epi) {
    case Epi::Store: return launch<BN, A_MN, B_MN, 0, CG>(g, s);
    case Epi::AddResidual: return launch<BN, A_MN, B_MN, 1, CG>(g, s);
    case Epi::AccumF32: return launch<BN, A_MN, B_MN, 2, CG>(g, s);
    case Epi::StoreGelu: return launch<BN, A_MN, B_MN, 3, CG>(g, s);
    case Epi::StoreF32: return launch<BN, A_MN, B_MN, 4, CG>(g, s);
    case Epi::MulGeluGrad: return launch<BN, A_MN, B_MN, 5, CG>(g, s);
    case Epi::Gelu: return launch<BN, A_MN, B_MN, 6, CG>(g, s);
  }
  return cudaErrorInvalidValue;
}

template <int BN, int CG>
cudaError_t launch_bn(const GemmArgs& g, cudaStream_t s) {
  const bool a_mn = !g.a_kmajor, b_mn = !g.b_kmajor;
  if (!a_mn && !b_mn) return launch_epi<BN, false, false, CG>(g, s);
  if (!a_mn && b_mn) return launch_epi<BN, false, true, CG>(g, s);
  if (a_mn && b_mn) return launch_epi<BN, true, true, CG>(g, s);
  return launch_epi<BN, true, false, CG>(g, s);
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.dt != DType::BF16) return false;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return false;
  if (g.M % BM || g.K % BK || g.N % 128) return false;
  const int ldc = g.ldc ? g.ldc : g.N;
  if (ldc % 8) return false;
  const uintptr_t align = reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B) |
                          reinterpret_cast<uintptr_t>(g.C) | reinterpret_cast<uintptr_t>(g.R) |
                          reinterpret_cast<uintptr_t>(g.G);
  if (align & 15) return false;
  return encode_fn() != nullptr;
}

cudaError_t gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (!gemm_tc_supported(g)) return cudaErrorInvalidValue;
  // CTA-pair (cta_group::2) tiles, 256 x 256 whenever N allows (measured:
  // smaller N tiles lose more per-tile efficiency than they win back in wave
  // quantisation).  M % 128 == 0 (supported): a half-empty last pair tile is
  // fine.
  if (g.N % 256 == 0) return launch_bn<256, 2>(g, s);
  if (g.N % 192 == 0 && g.b_kmajor) return launch_bn<192, 2>(g, s);
  return launch_bn<128, 2>(g, s);
}

}  // namespace gs
