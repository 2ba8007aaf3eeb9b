// tcgen05 GEMM for the complex64 contraction steps (K2 on the tensor cores).
//
// A complex GEMM C[M,N] = A[M,K] B[K,N] (the `np.tensordot` -> cgemm of
// tncut engine.py:129) is run as ONE real GEMM
//     C'[M][2N] = A'[M][2K] x B'^T,   A' = interleaved A,
//     B'[2n][2k..2k+1] = (br, -bi),  B'[2n+1][2k..2k+1] = (bi, br)
// whose fp32 output rows are exactly the interleaved complex64 rows of C.
// fp32 accuracy comes from a 2-term fp16 split with power-of-two scaling
// (x s = hi + lo): C' = Ahi Blo + Alo Bhi + Ahi Bhi, three kind::f16 UMMAs
// per K step.
//
// Structure (persistent, one CTA per SM; CG = 2 pairs two SMs on a 256-row
// tile with cta_group::2, each CTA staging its 128 rows of A and half of B):
//   warp 0    : TMA producer (4 tiles per stage: Ahi, Alo, Bhi, Blo), mbarrier ring
//   warp 1    : single-thread tcgen05.mma issuer (leader CTA only)
//   warp 2    : TMEM allocator (512 columns = 2 partial accumulators of 128 x 256 fp32)
//   warps 4-19: promotion + epilogue (TMEM partials -> fp32 registers -> global)
#include "tnb_internal.h"

#include <cuda.h>
#include <cstdlib>
#include <mutex>

#ifndef TNB_NB64_GROUPS
#define TNB_NB64_GROUPS 2
#endif

namespace tnb {
namespace {

constexpr int BM = 128;                      // rows per CTA
constexpr int BN = 256;                      // accumulator columns (fp32) of the widest tile
constexpr int BK = 32;                       // fp16 elements per stage row (64 B, SWIZZLE_64B)
constexpr int A_TILE = BM * BK * 2;          // 8 KB
constexpr int EPI_COLS = 64;                 // fp32 register accumulator columns per epilogue thread
// Tile width NB (accumulator columns): 256 for wide B operands; 128 / 64 for
// skinny ones (Np <= NB), whose 256-wide tiles were >= 75 % padding -- MMA,
// TMEM and epilogue work on columns that do not exist.  One epilogue warp
// group (4 lane quadrants) per 64 columns.
// Narrow tiles get more TMEM partial buffers (the MMA warp runs up to BUFS
// chunks ahead) and, at NB = 64, two epilogue groups that each own every
// other tile of the CTA unit: a short-K tile's epilogue is a latency chain
// (barrier wake-up, tcgen05.ld, stores), so two of them run concurrently.
template <int NB>
struct Epi {
  static constexpr int SPLIT = NB / EPI_COLS;     // column groups per TMEM lane quadrant
  static constexpr int GROUPS = NB == 64 ? TNB_NB64_GROUPS : 1; // tile-parallel epilogue groups (<= 384
                                                  // threads: the 64-float accumulators stay in registers)
  static constexpr int GROUP_THREADS = 128 * SPLIT;
  static constexpr int THREADS = GROUP_THREADS * GROUPS;  // epilogue threads
  static constexpr int NUM_THREADS = 128 + THREADS;
  static constexpr int BUFS = 512 / (GROUPS * NB);  // TMEM partial buffers per group (2-4)
  static_assert(BUFS * GROUPS * NB == 512, "TMEM columns");
};
constexpr int TMEM_COLS = 512;
constexpr int kDefaultChunkKb = 8;           // K blocks (of 32 fp16) per promotion chunk
constexpr int GROUP_M = 8;                   // rasterisation band height (m-tiles / CTA pairs)
constexpr int kDefaultPaceSlack = 32;        // K blocks a unit may run ahead of the slowest

template <int CG, int NB = BN>
struct Cfg {
  static constexpr int B_ROWS = NB / CG;                 // B rows staged by each CTA
  static constexpr int B_TILE = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
  // ring depth: ~192 KB of stages (6 at NB = 256; deeper for the narrow tiles,
  // whose short-K steps live on prefetch depth), 4 for single CTAs
  static constexpr int STAGES = CG == 1 ? 4 : (196608 / STAGE_BYTES > 10 ? 10 : 196608 / STAGE_BYTES);
  // narrow tiles stage the fused-store LUTs in shared memory; at NB = 256 the
  // extra 8 KB would push the carve-out to the 228 KB step and cost the wide
  // tiles ~12 % (measured), so they keep reading the LUTs through L1
  static constexpr int LUT_BYTES = NB < 256 ? 8192 : 0;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 512 /*barriers*/ + LUT_BYTES;
  static_assert((2 * STAGES + 2 * (512 / NB)) * 8 + 4 <= 512, "barrier area");
  // instruction descriptor: F32 accum, F16 x F16, K-major both, M = 128*CG, N = NB
  static constexpr uint32_t IDESC =
      (1u << 4) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}

// same, with a suspend-time hint: the waiting warp sleeps in hardware until
// the phase completes instead of re-polling (used for the long waits of the
// epilogue warps, which would otherwise keep issuing while the MMAs run)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(0x989680u)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// arrive on the same-offset barrier of CTA `rank` in the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

// Operands are K-blocked ([Kp/BK][rows][BK], see kKBlockLog): 3-D maps
// {BK, rows, K blocks}; a box {BK, rows, 1} is one contiguous tile.
template <int CG>
__device__ __forceinline__ void tma_load_tile(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                              int row, int kblock) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(0), "r"(row), "r"(kblock)
        : "memory");
  } else {
    // bytes land in this CTA's smem; completion is signalled on the LEADER's
    // barrier (peer bit of the shared::cluster address cleared)
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(0), "r"(row),
        "r"(kblock)
        : "memory");
  }
}

__device__ __forceinline__ uint64_t make_desc_sw64(const void* smem_ptr) {
  // K-major, SWIZZLE_64B: 8-row core groups 8*64 B apart (SBO), LBO unused.
  const uint64_t addr = smem_u32(smem_ptr);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;            // start address
  d |= (uint64_t)(512 >> 4) << 32;          // stride byte offset
  d |= 1ull << 46;                          // descriptor version (sm100)
  d |= 4ull << 61;                          // layout: SWIZZLE_64B
  return d;
}

template <int CG, int NB>
__device__ __forceinline__ void umma_f16(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t acc) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
        "l"(da), "l"(db), "r"(Cfg<1, NB>::IDESC), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
        "l"(da), "l"(db), "r"(Cfg<2, NB>::IDESC), "r"(acc));
  }
}

// MMA completion -> barrier(s): CG=1 own CTA; CG=2 the same barrier in both CTAs
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
  }
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t lut_lookup_s(const uint32_t (*t)[256], uint32_t j) {
  return t[0][j & 255] | t[1][(j >> 8) & 255] | t[2][(j >> 16) & 255] | t[3][j >> 24];
}

__device__ __forceinline__ uint32_t lut_lookup(const ByteLut* l, uint32_t j) {
  return __ldg(&l->t[0][j & 255]) | __ldg(&l->t[1][(j >> 8) & 255]) |
         __ldg(&l->t[2][(j >> 16) & 255]) | __ldg(&l->t[3][j >> 24]);
}

__device__ __forceinline__ void split2f(float a, float b, __half2& hi, __half2& lo) {
  hi = __floats2half2_rn(a, b);
  const float2 h = __half22float2(hi);
  lo = __floats2half2_rn(a - h.x, b - h.y);
}

// Fused staging store of one thread's 32 complex results (acc = interleaved
// re/im, already multiplied by alpha) into the consumer's operand layout:
// MODE 1 = rows operand (hi/lo of x s), MODE 2 = cols operand (rows 2n and
// 2n+1 of the 2x2 real expansion: (re, -im) and (im, re)), exactly what
// stage_kernel writes for a staged operand.
template <int MODE>
__device__ __forceinline__ void store_slot(const FuseOut& fo, uint32_t a, const float* x, float so) {
  // 4 consecutive complex (destination bits 0,1) -> 16-B hi/lo stores
  if constexpr (MODE == 1) {
    __half2 h[4], o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) split2f(x[2 * e] * so, x[2 * e + 1] * so, h[e], o[e]);
    *reinterpret_cast<uint4*>(fo.hi + a) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(fo.lo + a) = *reinterpret_cast<const uint4*>(o);
  } else {
    __half2 h0[4], o0[4], h1[4], o1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float re = x[2 * e] * so, im = x[2 * e + 1] * so;
      split2f(re, -im, h0[e], o0[e]);
      split2f(im, re, h1[e], o1[e]);
    }
    const uint32_t a1 = a + (1u << fo.L);
    *reinterpret_cast<uint4*>(fo.hi + a) = *reinterpret_cast<const uint4*>(h0);
    *reinterpret_cast<uint4*>(fo.lo + a) = *reinterpret_cast<const uint4*>(o0);
    *reinterpret_cast<uint4*>(fo.hi + a1) = *reinterpret_cast<const uint4*>(h1);
    *reinterpret_cast<uint4*>(fo.lo + a1) = *reinterpret_cast<const uint4*>(o1);
  }
}

// Fused staging store of one thread's 32 complex results (acc = interleaved
// re/im, already multiplied by alpha) into the consumer's operand layout:
// MODE 1 = rows operand (hi/lo of x s), MODE 2 = cols operand (rows 2n and
// 2n+1 of the 2x2 real expansion: (re, -im) and (im, re)), exactly what
// stage_kernel writes for a staged operand.  `tile` = destination of the
// warp's (row0, col0) corner.  `fast` is warp-uniform.
template <int MODE>
__device__ __forceinline__ void fused_store(const FuseOut& fo, const uint32_t (*lm)[256], uint32_t tile,
                                            float* acc, float so, int nvalid, int lane) {
  if (fo.fast && nvalid == 4 * fo.nslot) {
    // butterfly exchanges: slot q = complex 4q..4q+3 = floats 8q..8q+7
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int m = fo.xlane[j];
      if (m == 0) continue;
      const bool hi = (lane & m) != 0;
#pragma unroll
      for (int q0 = 0; q0 < 8; ++q0) {
        if (q0 & (1 << j)) continue;
        const int q1 = q0 | (1 << j);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float send = hi ? acc[8 * q0 + e] : acc[8 * q1 + e];
          const float recv = __shfl_xor_sync(0xffffffffu, send, m);
          if (hi) acc[8 * q0 + e] = recv; else acc[8 * q1 + e] = recv;
        }
      }
    }
    uint32_t a = tile;
#pragma unroll
    for (int b = 0; b < 5; ++b)
      if ((lane >> b) & 1) a |= fo.lane_w[b];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < fo.nslot) store_slot<MODE>(fo, a | fo.slot_w[q], acc + 8 * q, so);
  } else {
    const uint32_t base = tile | (lm != nullptr ? lut_lookup_s(lm, (uint32_t)lane)
                                                : lut_lookup(fo.lut_m, (uint32_t)lane));
#pragma unroll
    for (int j = 0; j < EPI_COLS / 2; ++j) {
      if (j >= nvalid) break;
      const uint32_t a = base | fo.dlow[j];
      const float re = acc[2 * j] * so, im = acc[2 * j + 1] * so;
      if constexpr (MODE == 1) {
        __half2 h, o;
        split2f(re, im, h, o);
        fo.hi[a] = h;
        fo.lo[a] = o;
      } else {
        __half2 h0, o0, h1, o1;
        split2f(re, -im, h0, o0);
        split2f(im, re, h1, o1);
        const uint32_t a1 = a + (1u << fo.L);
        fo.hi[a] = h0; fo.lo[a] = o0;
        fo.hi[a1] = h1; fo.lo[a1] = o1;
      }
    }
  }
}

struct WorkCoord {
  int split, mb, nb;
};

// Grouped raster: bands of group_m m-tiles, m fastest inside a band, then n.
// The tiles in flight then cover ~16 m-tiles x ~9 n-tiles, so each A panel
// (rows x K) and B panel streamed from HBM is shared through L2 by the
// concurrently running CTAs.
__device__ __forceinline__ WorkCoord decode(int w, int nm, int nn, int group_m) {
  const int per_split = nm * nn;
  WorkCoord c;
  c.split = w / per_split;
  const int t = w - c.split * per_split;
  const int band = t / (group_m * nn);
  const int idx = t - band * (group_m * nn);
  const int band_m = min(group_m, nm - band * group_m);
  c.mb = band * group_m + idx % band_m;
  c.nb = idx / band_m;
  return c;
}

// Accumulation: the tensor cores' fp32 accumulator loses precision over
// thousands of K steps (measured ~15x the IEEE fp32 error growth).  K is
// therefore processed in chunks of `chunk_kb` K blocks into one of two TMEM
// partial accumulators; the epilogue warps promote every finished partial
// into an IEEE fp32 register accumulator (DeepGEMM-style promotion), while
// the MMA warp fills the other partial.
template <int CG, int NB>
__global__ void __launch_bounds__(Epi<NB>::NUM_THREADS, 1)
gemm_f16x3_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                  const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                  float* __restrict__ C, int M, int Np, int Kp, int splits, int k_per_split,
                  int chunk_kb, int group_m, const ScaleSrc scale_rows, const ScaleSrc scale_cols,
                  unsigned int* __restrict__ max_out, unsigned int* __restrict__ progress,
                  int pace_slack, const __grid_constant__ FuseOut fo, int epi_spin) {
  using CF = Cfg<CG, NB>;
  constexpr int STAGES = CF::STAGES;
  // fp16 scale-guard re-run of a fused producer: nothing to do unless the
  // guard fires (same decision in every CTA, before any barrier or TMEM use)
  if (fo.redo && !fused_redo_fires(fo)) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  // TMEM partial accumulators: as many NB-column buffers as the 512 columns
  // hold (2 at NB = 256, 8 at NB = 64), so the MMA warp can run NBUF chunks
  // ahead of the epilogue -- short-K tiles (one or two K blocks) are then no
  // longer serialised on the epilogue's TMEM read latency
  constexpr int NBUF = TMEM_COLS / NB;
  constexpr int GROUPS = Epi<NB>::GROUPS, BUFS = Epi<NB>::BUFS;
  uint64_t* pfull_bar = empty_bar + STAGES;
  uint64_t* pempty_bar = pfull_bar + NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty_bar + NBUF);
  // fused-store destination LUTs (rows, cols) staged in shared memory
  uint32_t (*lut_s)[4][256] = reinterpret_cast<uint32_t (*)[4][256]>(
      smem + STAGES * CF::STAGE_BYTES + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 1 ? 0u : cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG;       // tile-processing unit (CTA or CTA pair)
  const int n_units = gridDim.x / CG;
  const int nm = (M + BM * CG - 1) / (BM * CG);
  const int nn = (Np + NB - 1) / NB;
  const int total = nm * nn * splits;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_blo)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], CG);          // leader: own arrive(+tx) and the peer's arrive
      mbar_init(&empty_bar[i], 1);          // MMA commit (multicast to both CTAs)
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&pfull_bar[i], 1);          // MMA commit (multicast)
      mbar_init(&pempty_bar[i], CG * Epi<NB>::GROUP_THREADS);  // leader: one epilogue group of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (CF::LUT_BYTES > 0 && fo.mode != 0 && warp >= 4) {
    for (int i = threadIdx.x - 128; i < 2048; i += Epi<NB>::THREADS) {
      const ByteLut* l = i < 1024 ? fo.lut_m : fo.lut_n;
      const int j = i & 1023;
      lut_s[i >> 10][j >> 8][j & 255] = __ldg(&l->t[j >> 8][j & 255]);
    }
  }
  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (both CTAs; lane 0 issues, the warp helps pacing) =====
    // Soft pacing (leader): every unit publishes its K-block count; a unit
    // more than `pace_slack` blocks ahead of the slowest one waits, so the
    // CTAs streaming the same A/B panels stay within the L2 reuse window.
    int stage = 0;
    uint32_t phase = 0;
    uint32_t issued = 0;
    const bool pace = pace_slack > 0 && leader && progress != nullptr;
    for (int w = unit; w < total; w += n_units) {
      const WorkCoord wc = decode(w, nm, nn, group_m);
      const int k_begin = wc.split * k_per_split;
      const int k_end = min(Kp, k_begin + k_per_split);
      const int m0 = wc.mb * BM * CG + (int)rank * BM;
      const int n0 = wc.nb * NB + (int)rank * CF::B_ROWS;
      for (int k = k_begin; k < k_end; k += BK, ++issued) {
        if (pace && (issued & 15) == 0) {
          if (lane == 0) atomicExch(progress + unit, issued);
          for (;;) {
            unsigned int mn = 0xFFFFFFFFu;
            for (int u = lane; u < n_units; u += 32) mn = min(mn, __ldcg(progress + u));
            mn = __reduce_min_sync(0xffffffffu, mn);
            if (mn == 0xFFFFFFFFu || issued <= mn + (unsigned)pace_slack) break;
            __nanosleep(128);
          }
        }
        if (lane == 0) {
          if (epi_spin & 4) mbar_wait(&empty_bar[stage], phase ^ 1);
          else mbar_wait_sleep(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * CF::STAGE_BYTES;
          const int kbk = k / BK;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], CG * (2 * A_TILE + 2 * CF::B_TILE));
          else mbar_arrive_remote(&full_bar[stage], 0);
          tma_load_tile<CG>(st, &tm_ahi, &full_bar[stage], m0, kbk);
          tma_load_tile<CG>(st + A_TILE, &tm_alo, &full_bar[stage], m0, kbk);
          tma_load_tile<CG>(st + 2 * A_TILE, &tm_bhi, &full_bar[stage], n0, kbk);
          tma_load_tile<CG>(st + 2 * A_TILE + CF::B_TILE, &tm_blo, &full_bar[stage], n0, kbk);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    if (pace && lane == 0) atomicExch(progress + unit, 0xFFFFFFFFu);  // done: never hold others back
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (leader CTA) =====
      int stage = 0;
      uint32_t phase = 0;
      int gcnt[GROUPS];
#pragma unroll
      for (int g = 0; g < GROUPS; ++g) gcnt[g] = 0;
      int tseq = 0;
      for (int w = unit; w < total; w += n_units, ++tseq) {
        const WorkCoord wc = decode(w, nm, nn, group_m);
        const int k_begin = wc.split * k_per_split;
        const int nkb = (min(Kp, k_begin + k_per_split) - k_begin + BK - 1) / BK;
        const int g = tseq % GROUPS;  // the epilogue group that owns this tile
        int gc = 0;
#pragma unroll
        for (int x = 0; x < GROUPS; ++x) if (x == g) gc = gcnt[x];
        for (int c0 = 0; c0 < nkb; c0 += chunk_kb, ++gc) {
          const int buf = g * BUFS + gc % BUFS;
          const uint32_t par = (uint32_t)(gc / BUFS) & 1u;
          if (epi_spin & 2) mbar_wait(&pempty_bar[buf], par ^ 1);
          else mbar_wait_sleep(&pempty_bar[buf], par ^ 1);
          tc_fence_after();
          const uint32_t tmem_c = tmem_base + buf * NB;
          const int c1 = min(nkb, c0 + chunk_kb);
          for (int kb = c0; kb < c1; ++kb) {
            if (epi_spin & 2) mbar_wait(&full_bar[stage], phase);
            else mbar_wait_sleep(&full_bar[stage], phase);
            tc_fence_after();
            if (lane == 0) {
              uint8_t* st = smem + stage * CF::STAGE_BYTES;
              const uint64_t d_ahi = make_desc_sw64(st);
              const uint64_t d_alo = make_desc_sw64(st + A_TILE);
              const uint64_t d_bhi = make_desc_sw64(st + 2 * A_TILE);
              const uint64_t d_blo = make_desc_sw64(st + 2 * A_TILE + CF::B_TILE);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 16 fp16 = 32 B along K
                umma_f16<CG, NB>(tmem_c, d_ahi + adv, d_blo + adv, (kb == c0 && kk == 0) ? 0u : 1u);
                umma_f16<CG, NB>(tmem_c, d_alo + adv, d_bhi + adv, 1u);
                umma_f16<CG, NB>(tmem_c, d_ahi + adv, d_bhi + adv, 1u);
              }
              umma_commit<CG>(&empty_bar[stage]);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (lane == 0) umma_commit<CG>(&pfull_bar[buf]);
          __syncwarp();
        }
#pragma unroll
        for (int x = 0; x < GROUPS; ++x) if (x == g) gcnt[x] = gc;
      }
    }
  } else if (warp >= 4) {
    // ===== promotion + epilogue: warp -> TMEM lane quadrant (warp % 4), column group =====
    const int q = warp & 3;
    const int grp = ((warp - 4) >> 2) % Epi<NB>::SPLIT;   // column group
    const int eg = ((warp - 4) >> 2) / Epi<NB>::SPLIT;    // epilogue group (tiles tseq % GROUPS == eg)
    const float alpha =
        splits == 1 ? 1.f / (scale_from_src(scale_rows) * scale_from_src(scale_cols)) : 1.f;
    const float so = fo.mode != 0 ? scale_from_src(fo.scale) : 1.f;  // fused: consumer's scale
    float vmax = 0.f;  // max |C| of this thread's outputs (scale slot of the result tensor)
    int gc = 0;         // chunks of this group's tiles so far
    int tseq = 0;
    for (int w = unit; w < total; w += n_units, ++tseq) {
      if (tseq % GROUPS != eg) continue;
      const WorkCoord wc = decode(w, nm, nn, group_m);
      const int k_begin = wc.split * k_per_split;
      const int nkb = (min(Kp, k_begin + k_per_split) - k_begin + BK - 1) / BK;
      float acc[EPI_COLS];
#pragma unroll
      for (int j = 0; j < EPI_COLS; ++j) acc[j] = 0.f;
      for (int c0 = 0; c0 < nkb; c0 += chunk_kb, ++gc) {
        const int buf = eg * BUFS + gc % BUFS;
        const uint32_t par = (uint32_t)(gc / BUFS) & 1u;
        if (epi_spin & 1) mbar_wait(&pfull_bar[buf], par);
        else mbar_wait_sleep(&pfull_bar[buf], par);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * NB + grp * EPI_COLS;
#pragma unroll
        for (int s = 0; s < EPI_COLS / 16; ++s) {
          uint32_t r[16];
          tmem_ld16(taddr + s * 16, r);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[s * 16 + j] += __uint_as_float(r[j]);
        }
        tc_fence_before();
        if (CG == 1 || leader) mbar_arrive(&pempty_bar[buf]);
        else mbar_arrive_remote(&pempty_bar[buf], 0);
      }
      const int row0 = wc.mb * BM * CG + (int)rank * BM + q * 32;
      const int row = row0 + lane;
      const int col0 = wc.nb * NB + grp * EPI_COLS;
      {
        // max |C| of the tile (alpha > 0 is a power of two: max|x alpha| = alpha max|x|)
        float tm = 0.f;
#pragma unroll
        for (int j = 0; j < EPI_COLS; ++j) tm = fmaxf(tm, fabsf(acc[j]));  // out-of-range rows/cols are TMA zero-fill
        vmax = fmaxf(vmax, tm * alpha);
      }
      if (fo.mode == 0) {
#pragma unroll
        for (int j = 0; j < EPI_COLS; ++j) acc[j] *= alpha;
      }
      if (fo.mode != 0) {
        // fused staging: write the consumer's fp16 operand directly
        const int nvalid = min(EPI_COLS / 2, (Np - col0) >> 1);
        if (nvalid > 0) {  // warp-uniform; every row of a 32-row group exists (M >= 128, 2^k)
          const uint32_t tile = CF::LUT_BYTES > 0
              ? lut_lookup_s(lut_s[0], (uint32_t)row0) | lut_lookup_s(lut_s[1], (uint32_t)(col0 >> 1))
              : lut_lookup(fo.lut_m, (uint32_t)row0) | lut_lookup(fo.lut_n, (uint32_t)(col0 >> 1));
          // (x alpha) so == x (alpha so) exactly: both are powers of two
          const uint32_t (*lm)[256] = CF::LUT_BYTES > 0 ? lut_s[0] : nullptr;
          if (fo.mode == 1) fused_store<1>(fo, lm, tile, acc, alpha * so, nvalid, lane);
          else fused_store<2>(fo, lm, tile, acc, alpha * so, nvalid, lane);
        }
      } else if (row0 + 32 <= M && col0 + EPI_COLS <= Np) {
        // full 32-row x 64-column block: transpose float4 chunks inside each
        // 8-lane group (3 xor-butterfly stages) so that every store writes
        // 4 rows x 128 contiguous bytes instead of 32 rows x 16 bytes
        const int g8 = lane & 7;
        float* base = C + (size_t)wc.split * (size_t)M * (size_t)Np + (size_t)(row0 + (lane & ~7)) * Np + col0;
#pragma unroll
        for (int b = 0; b < EPI_COLS / 32; ++b) {
          float* x = acc + b * 32;  // 8 float4 chunks: chunk c = x[4c..4c+3]
#pragma unroll
          for (int m = 4; m > 0; m >>= 1) {
            const bool hi = (g8 & m) != 0;
#pragma unroll
            for (int c0 = 0; c0 < 8; ++c0) {
              if (c0 & m) continue;
              const int c1 = c0 | m;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float send = hi ? x[4 * c0 + e] : x[4 * c1 + e];
                const float recv = __shfl_xor_sync(0xffffffffu, send, m);
                if (hi) x[4 * c0 + e] = recv; else x[4 * c1 + e] = recv;
              }
            }
          }
          // x chunk s now holds chunk g8 of row (lane & ~7) + s
#pragma unroll
          for (int s = 0; s < 8; ++s)
            *reinterpret_cast<float4*>(base + (size_t)s * Np + b * 32 + 4 * g8) =
                make_float4(x[4 * s], x[4 * s + 1], x[4 * s + 2], x[4 * s + 3]);
        }
      } else if (row < M && col0 < Np) {
        float* dst = C + (size_t)wc.split * (size_t)M * (size_t)Np + (size_t)row * Np + col0;
        if (col0 + EPI_COLS <= Np) {
#pragma unroll
          for (int j = 0; j < EPI_COLS; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else if (((Np - col0) & 3) == 0) {  // skinny B: the valid columns in 16-B stores
#pragma unroll
          for (int j = 0; j < EPI_COLS; j += 4)
            if (col0 + j < Np)
              *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < EPI_COLS; ++j)
            if (col0 + j < Np) dst[j] = acc[j];
        }
      }
    }
    if (splits == 1 && max_out != nullptr) {
      for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
      if (lane == 0 && vmax > 0.f) atomicMax(max_out, __float_as_uint(vmax));
    }
  }

  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Host side: tensor maps through the driver entry point (no -lcuda needed).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw Error(TNB_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  return fn;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

void make_map(void* out, const __half* base, int64_t rows, int64_t kp, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (kp % 8) != 0)
    throw Error(TNB_ERR_SHAPE, "tensor-core operand not 16-byte aligned");
  // K-blocked layout [kp/BK][rows][BK] (plain [rows][kp] when kp <= BK)
  static_assert(BK == 2 << kKBlockLog, "GEMM K block must match the staging block");
  const int64_t inner = kp < BK ? kp : BK;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)(kp / inner)};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)(inner * 2 * rows)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  static const int promo_env = env_int("TNB_L2_PROMO", -1);
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (promo_env == 0) promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  if (promo_env == 64) promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  if (promo_env == 128) promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  CUresult r = get_encode()(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                            const_cast<__half*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, promo,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(TNB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// CTA group for a GEMM: pairs (cta_group::2) whenever the rows fill 256-row tiles
int choose_cg(int64_t M) {
  static const int forced = env_int("TNB_CTA_GROUP", 0);
  if (forced == 1 || forced == 2) return forced;
  return M >= 256 ? 2 : 1;
}

// tile width: the narrowest of 64 / 128 / 256 that holds the B operand's
// columns (TNB_GEMM_NB forces one; 0 = auto)
int choose_nb(int64_t Np) {
  static const int forced = env_int("TNB_GEMM_NB", 0);
  if (forced == 64 || forced == 128 || forced == 256) return forced;
  return Np <= 64 ? 64 : (Np <= 128 ? 128 : 256);
}

int choose_splits(int64_t M, int64_t Np, int64_t Kp, int num_sms) {
  static const int no_split = env_int("TNB_NO_SPLITK", 0);
  if (no_split) return 1;
  const int cg = choose_cg(M);
  const int nb = choose_nb(Np);
  const int64_t units = num_sms / cg;
  const int64_t tiles = ((M + BM * cg - 1) / (BM * cg)) * ((Np + nb - 1) / nb);
  const int64_t kblocks = (Kp + BK - 1) / BK;
  // split K when the tiles leave CTA units idle: as many splits as fill the
  // units (any count, not only powers of two), each keeping >= 16 K blocks
  if (tiles * 2 > units) return 1;
  int64_t s = units / tiles;
  s = std::min<int64_t>(s, kblocks / 16);
  s = std::min<int64_t>(s, 64);
  return (int)std::max<int64_t>(s, 1);
}

}  // namespace

bool tc_available(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return false;
  return prop.major == 10 && prop.minor == 0;
}

int tc_splits(int64_t M, int64_t Np, int64_t Kp, int num_sms) {
  return choose_splits(M, Np, Kp, num_sms);
}

int64_t tc_workspace_elems(int64_t M, int64_t Np, int64_t Kp, int num_sms) {
  const int s = choose_splits(M, Np, Kp, num_sms);
  return s > 1 ? (int64_t)s * M * Np : 0;
}

void tc_plan_gemm(TcGemmPlan* p, const __half* Ahi, const __half* Alo, const __half* Bhi,
                  const __half* Blo, int64_t M, int64_t Np, int64_t Kp, float* C, float* workspace,
                  int64_t workspace_elems, const ScaleSrc& scale_rows,
                  const ScaleSrc& scale_cols, unsigned int* max_out, int num_sms) {
  if (M > (1ll << 31) - 1 || Np > (1ll << 31) - 1 || Kp > (1ll << 31) - 1)
    throw Error(TNB_ERR_SHAPE, "tensor-core GEMM dimension too large");
  p->M = M; p->Np = Np; p->Kp = Kp;
  p->cta_group = choose_cg(M);
  p->nb = choose_nb(Np);
  p->splits = choose_splits(M, Np, Kp, num_sms);
  const int64_t kblocks = (Kp + BK - 1) / BK;
  p->k_per_split = ((kblocks + p->splits - 1) / p->splits) * BK;
  static const int max_sms = env_int("TNB_GEMM_MAX_SMS", 0);  // diagnostic: cap the persistent grid
  const int64_t units = (max_sms > 0 && max_sms < num_sms ? max_sms : num_sms) / p->cta_group;
  const int64_t work = ((M + BM * p->cta_group - 1) / (BM * p->cta_group)) * ((Np + p->nb - 1) / p->nb) * p->splits;
  p->grid = (int)((work < units ? work : units) * p->cta_group);
  if (p->splits > 1) {
    if (workspace == nullptr || workspace_elems < (int64_t)p->splits * M * Np)
      throw Error(TNB_ERR_ARG, "split-K workspace too small");
    p->C = workspace;
  } else {
    p->C = C;
  }
  p->scale_rows = scale_rows;
  p->scale_cols = scale_cols;
  p->max_out = max_out;
  // promotion chunk: always on (the tensor cores' long-K accumulation error is
  // ~15x IEEE fp32, profiles/r1/gemm_accuracy_vs_promotion_chunk.txt)
  p->chunk_kb = env_int("TNB_CHUNK_KB", kDefaultChunkKb);
  if (p->chunk_kb <= 0 || p->chunk_kb > 64) p->chunk_kb = kDefaultChunkKb;
  p->group_m = env_int("TNB_GROUP_M", GROUP_M);
  if (p->group_m <= 0) p->group_m = 1 << 30;
  // soft pacing keeps long-K tiles inside the L2 window (top C4 GEMM: 75 vs
  // 343 GB DRAM without it); tiles of few K blocks turn over fast enough for
  // the raster alone, and there the lockstep costs 6-8% of the cycles
  static const int pace_min_kb = env_int("TNB_PACE_MIN_KB", 64);
  // ... and only when the smaller operand does not sit in L2 anyway (a few-MB
  // B panel is shared by every tile without help)
  static const int pace_min_mb = env_int("TNB_PACE_MIN_MB", 0);
  const double small_mb = (double)std::min(M, Np) * (double)Kp * 4.0 / 1048576.0;
  p->pace_slack = kblocks / p->splits >= pace_min_kb && small_mb >= pace_min_mb
                      ? env_int("TNB_PACE", kDefaultPaceSlack) : 0;
  static const int spin = env_int("TNB_EPI_SPIN", -1);
  p->epi_spin = spin >= 0 ? spin : 0;
  const int b_rows = p->nb / p->cta_group;
  p->ahi = Ahi; p->alo = Alo; p->bhi = Bhi; p->blo = Blo;
  // short-K skinny steps (one K block of <= 32 real, <= 64 real columns):
  // per 256-row tile the tcgen05 pipeline is a latency chain (TMA -> MMA ->
  // TMEM -> epilogue, ~1.6 us per tile at M = 2^23, N = 16, K = 8 complex);
  // the same staged operands through the FP32 pipe stream at HBM speed
  static const int skinny_env = env_int("TNB_SKINNY", 1);
  // (from M = 2^22 rows: at 2^20 the tcgen05 path's 4096 tiles still beat
  // the FP32 kernel, 0.105 vs 0.158 ms measured)
  p->skinny = skinny_env && Kp <= 32 && Np <= 64 && p->splits == 1 && M >= (1 << 22);
  make_map(p->tmap[0], Ahi, M, Kp, BM);
  make_map(p->tmap[1], Alo, M, Kp, BM);
  make_map(p->tmap[2], Bhi, Np, Kp, b_rows);
  make_map(p->tmap[3], Blo, Np, Kp, b_rows);
}

template <int CG, int NB>
void launch_cg(const TcGemmPlan* p, cudaStream_t s) {
  auto kern = gemm_f16x3_kernel<CG, NB>;
  TNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<CG, NB>::SMEM_BYTES));
  const CUtensorMap* maps = reinterpret_cast<const CUtensorMap*>(p->tmap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->grid);
  cfg.blockDim = dim3(Epi<NB>::NUM_THREADS);
  cfg.dynamicSmemBytes = Cfg<CG, NB>::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p->progress && p->pace_slack > 0)
    TNB_CUDA(cudaMemsetAsync(p->progress, 0, sizeof(unsigned int) * (p->grid / CG), s));
  TNB_CUDA(cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], p->C, (int)p->M,
                              (int)p->Np, (int)p->Kp, p->splits, (int)p->k_per_split, p->chunk_kb,
                              p->group_m, p->scale_rows, p->scale_cols, p->max_out, p->progress,
                              p->pace_slack, p->fuse, p->epi_spin));
}

// Short-K skinny GEMM on the FP32 pipe (TcGemmPlan::skinny): C'[m][0..Np)
// = alpha * sum_k (Ahi + Alo)[m][k] (Bhi + Blo)[n][k] over the SAME staged
// operands and with the SAME epilogue (fused staged store or fp32 C, max
// publication, scale-guard re-run prologue) as gemm_f16x3_kernel.  Kp <= 32
// means the staged layouts are plain [rows][Kp] (one K block).  One thread
// per row, warps on 32 consecutive rows (the fused store's lane mapping).
template <int KP, int NP>
__global__ void __launch_bounds__(256)
gemm_skinny_kernel(const __half* __restrict__ ahi, const __half* __restrict__ alo,
                   const __half* __restrict__ bhi, const __half* __restrict__ blo,
                   float* __restrict__ C, int64_t M, const ScaleSrc scale_rows,
                   const ScaleSrc scale_cols, unsigned int* __restrict__ max_out,
                   const __grid_constant__ FuseOut fo) {
  if (fo.redo && !fused_redo_fires(fo)) return;
  __shared__ float bs[NP][KP + 1];
  for (int i = threadIdx.x; i < NP * KP; i += blockDim.x) {
    const int n = i / KP, k = i % KP;
    bs[n][k] = __half2float(bhi[i]) + __half2float(blo[i]);
  }
  const float alpha = 1.f / (scale_from_src(scale_rows) * scale_from_src(scale_cols));
  const float so = fo.mode != 0 ? scale_from_src(fo.scale) : 1.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float vmax = 0.f;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < M;
       row += (int64_t)gridDim.x * blockDim.x) {
    float a[KP];
#pragma unroll
    for (int k = 0; k < KP; k += 8) {
      const uint4 h = *reinterpret_cast<const uint4*>(ahi + row * KP + k);
      const uint4 l = *reinterpret_cast<const uint4*>(alo + row * KP + k);
      const __half2* hh = reinterpret_cast<const __half2*>(&h);
      const __half2* ll = reinterpret_cast<const __half2*>(&l);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __half22float2(hh[e]), y = __half22float2(ll[e]);
        a[k + 2 * e] = x.x + y.x;
        a[k + 2 * e + 1] = x.y + y.y;
      }
    }
    float acc[EPI_COLS];
#pragma unroll
    for (int n = 0; n < EPI_COLS; ++n) {
      float v = 0.f;
      if (n < NP) {
#pragma unroll
        for (int k = 0; k < KP; ++k) v = fmaf(a[k], bs[n][k], v);
      }
      acc[n] = v;
    }
    float tm = 0.f;
#pragma unroll
    for (int n = 0; n < NP; ++n) tm = fmaxf(tm, fabsf(acc[n]));
    vmax = fmaxf(vmax, tm * alpha);
    if (fo.mode != 0) {
      const int64_t row0 = row & ~(int64_t)31;
      // LUTs through L1 (every block staging them into shared memory measured
      // 1.75x slower: 2368 blocks x 8 KB of setup)
      const uint32_t tile = lut_lookup(fo.lut_m, (uint32_t)row0) | lut_lookup(fo.lut_n, 0u);
      if (fo.mode == 1) fused_store<1>(fo, nullptr, tile, acc, alpha * so, NP / 2, lane);
      else fused_store<2>(fo, nullptr, tile, acc, alpha * so, NP / 2, lane);
    } else {
      float* dst = C + row * NP;
#pragma unroll
      for (int n = 0; n < NP; n += 4)
        *reinterpret_cast<float4*>(dst + n) =
            make_float4(acc[n] * alpha, acc[n + 1] * alpha, acc[n + 2] * alpha, acc[n + 3] * alpha);
    }
  }
  if (max_out != nullptr) {
    for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if (lane == 0 && vmax > 0.f) atomicMax(max_out, __float_as_uint(vmax));
  }
}

template <int KP, int NP>
void launch_skinny(const TcGemmPlan* p, cudaStream_t s) {
  int64_t blocks = (p->M + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gemm_skinny_kernel<KP, NP><<<(unsigned)blocks, 256, 0, s>>>(
      p->ahi, p->alo, p->bhi, p->blo, p->C, p->M, p->scale_rows, p->scale_cols, p->max_out, p->fuse);
}

void tc_launch_gemm(const TcGemmPlan* p, cudaStream_t s) {
  if (p->skinny) {
    const int key = (int)p->Kp * 1000 + (int)p->Np;
    switch (key) {
      case 8008: launch_skinny<8, 8>(p, s); break;
      case 8016: launch_skinny<8, 16>(p, s); break;
      case 8032: launch_skinny<8, 32>(p, s); break;
      case 8064: launch_skinny<8, 64>(p, s); break;
      case 16008: launch_skinny<16, 8>(p, s); break;
      case 16016: launch_skinny<16, 16>(p, s); break;
      case 16032: launch_skinny<16, 32>(p, s); break;
      case 16064: launch_skinny<16, 64>(p, s); break;
      case 32008: launch_skinny<32, 8>(p, s); break;
      case 32016: launch_skinny<32, 16>(p, s); break;
      case 32032: launch_skinny<32, 32>(p, s); break;
      case 32064: launch_skinny<32, 64>(p, s); break;
      default: throw Error(TNB_ERR_ARG, "unsupported skinny GEMM shape");
    }
    check_launch("gemm_skinny");
    return;
  }
  const int key = p->cta_group * 1000 + p->nb;
  switch (key) {
    case 2256: launch_cg<2, 256>(p, s); break;
    case 2128: launch_cg<2, 128>(p, s); break;
    case 2064: launch_cg<2, 64>(p, s); break;
    case 1256: launch_cg<1, 256>(p, s); break;
    case 1128: launch_cg<1, 128>(p, s); break;
    case 1064: launch_cg<1, 64>(p, s); break;
    default: throw Error(TNB_ERR_ARG, "unsupported GEMM tile configuration");
  }
  check_launch("gemm_f16x3");
}

}  // namespace tnb
