// SIMT kernels of the executor: sliced-leaf gather (K1), generic gathered
// complex contraction for small steps (K2/K3 below the tensor-core
// threshold), bit-permutation (K4), deterministic slice-sum accumulator
// (K5), and the operand staging for the tcgen05 3xFP16 path.
//
// Reference call sites replaced (tncut engine.py): `_prepared_leaves`
// :102-114 (np.take per sliced axis), `np.tensordot` / `np.multiply.outer`
// :125-131, root transpose :287-290, `_fixed_tree_sum` :207-222.
#include "tnb_internal.h"

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace tnb {

namespace {

constexpr int kSms = 148;
// staging tiles: 2^kStageTileBits elements; contiguous runs of 2^kStageRunBits
// elements on both the source (reads) and the destination (writes) side
int stage_tile_bits() {
  static const int v = [] { const char* e = getenv("TNB_STAGE_TILE"); int x = e ? atoi(e) : 11; return x < 8 ? 8 : (x > 12 ? 12 : x); }();
  return v;
}
int stage_run_bits() {
  static const int v = [] { const char* e = getenv("TNB_STAGE_RUN"); int x = e ? atoi(e) : 5; return x < 3 ? 3 : (x > 7 ? 7 : x); }();
  return v;
}

__device__ __forceinline__ uint32_t lut_map(const uint32_t (*t)[256], uint32_t j) {
  return t[0][j & 255u] | t[1][(j >> 8) & 255u] | t[2][(j >> 16) & 255u] | t[3][j >> 24];
}

template <typename T> struct Scalar;
template <> struct Scalar<float2> { using type = float; };
template <> struct Scalar<double2> { using type = double; };

template <typename T>
__device__ __forceinline__ T cadd(T a, T b) { T r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }

// block-wide max of non-negative floats -> one atomicMax on the bit pattern
__device__ __forceinline__ void block_max_atomic(float m, unsigned int* out) {
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
  }
}


// ---------------------------------------------------------------------------
// K1: sliced-leaf preparation.  One block per sliced leaf; the selected
// sub-tensor for this mask is gathered into the slice pool.
template <typename T>
__global__ void prepare_leaves_kernel(const T* __restrict__ pool, T* __restrict__ out,
                                      const SlicedLeafDesc* __restrict__ descs,
                                      const uint32_t* __restrict__ keep, uint64_t mask) {
  const SlicedLeafDesc d = descs[blockIdx.x];
  uint64_t base = d.src_off;
  for (uint32_t i = 0; i < d.n_sl; ++i)
    if ((mask >> d.sl_bit[i]) & 1ull) base += d.sl_stride[i];
  for (uint32_t j = threadIdx.x; j < d.out_elems; j += blockDim.x)
    out[d.dst_off + j] = pool[base + keep[d.keep_lut_off + j]];
}

// ---------------------------------------------------------------------------
// Gathered SIMT contraction: C[m*N+n] = sum_k A[lutA(m*K+k)] * B[lutB(n*K+k)].
// 32x32 output tile per 256-thread block, 2x2 per thread, K chunks of 16.
// `tile` = this block's tile index within the step.
template <typename T>
__device__ __forceinline__ void simt_tile(const T* __restrict__ A, const T* __restrict__ B,
                                          T* __restrict__ C, int64_t M, int64_t N, int64_t K,
                                          const ByteLut* __restrict__ gla,
                                          const ByteLut* __restrict__ glb,
                                          unsigned int* __restrict__ max_out, int64_t tile) {
  using S = typename Scalar<T>::type;
  constexpr int BM = 32, BN = 32, BK = 16;
  __shared__ uint32_t la[4][256];
  __shared__ uint32_t lb[4][256];
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += 256) {
    la[i >> 8][i & 255] = gla->t[i >> 8][i & 255];
    lb[i >> 8][i & 255] = glb->t[i >> 8][i & 255];
  }
  const int64_t nbn = (N + BN - 1) / BN;
  const int64_t m0 = (tile / nbn) * BM, n0 = (tile % nbn) * BN;
  const int tx = tid & 15, ty = tid >> 4;
  S acc_re[2][2] = {{0, 0}, {0, 0}}, acc_im[2][2] = {{0, 0}, {0, 0}};
  __syncthreads();
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    for (int i = tid; i < BM * BK; i += 256) {
      const int mm = i / BK, kk = i % BK;
      const int64_t m = m0 + mm, k = k0 + kk;
      T v; v.x = 0; v.y = 0;
      if (m < M && k < K) v = A[lut_map(la, (uint32_t)(m * K + k))];
      As[kk][mm] = v;
    }
    for (int i = tid; i < BN * BK; i += 256) {
      const int nn = i / BK, kk = i % BK;
      const int64_t n = n0 + nn, k = k0 + kk;
      T v; v.x = 0; v.y = 0;
      if (n < N && k < K) v = B[lut_map(lb, (uint32_t)(n * K + k))];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a0 = As[kk][ty], a1 = As[kk][ty + 16];
      T b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
      const T av[2] = {a0, a1};
      const T bv[2] = {b0, b1};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          acc_re[i][j] += av[i].x * bv[j].x - av[i].y * bv[j].y;
          acc_im[i][j] += av[i].x * bv[j].y + av[i].y * bv[j].x;
        }
    }
    __syncthreads();
  }
  float vmax = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        T v; v.x = acc_re[i][j]; v.y = acc_im[i][j];
        C[m * N + n] = v;
        vmax = fmaxf(vmax, (float)fmax(fabs(v.x), fabs(v.y)));
      }
    }
  if (max_out) block_max_atomic(vmax, max_out);
}

// Wide tiles for big SIMT steps (the fp64 path): 64x64 outputs per block,
// 4x4 per thread, K in blocks of 16 staged through shared memory with the
// same LUT gathers as simt_tile.  Four times the FMAs per shared-memory load
// of the 32x32 tile (2 vs 0.5 flop/B), so the big complex128 GEMMs of a slice
// run on the FP64 pipe instead of shared-memory bandwidth.
template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 16 ? 1 : 2)
contract_wide_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                     int64_t M, int64_t N, int64_t K, const ByteLut* __restrict__ gla,
                     const ByteLut* __restrict__ glb, unsigned int* __restrict__ max_out) {
  using S = typename Scalar<T>::type;
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ uint32_t la[4][256];
  __shared__ uint32_t lb[4][256];
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += 256) {
    la[i >> 8][i & 255] = gla->t[i >> 8][i & 255];
    lb[i >> 8][i & 255] = glb->t[i >> 8][i & 255];
  }
  const int64_t nbn = (N + BN - 1) / BN;
  const int64_t m0 = ((int64_t)blockIdx.x / nbn) * BM, n0 = ((int64_t)blockIdx.x % nbn) * BN;
  const int tx = tid & 15, ty = tid >> 4;
  S acc_re[4][4], acc_im[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc_re[i][j] = acc_im[i][j] = 0;
  __syncthreads();
  // software pipeline: the gathers of K block k0 + BK are in flight (in
  // registers) while block k0 is multiplied out of shared memory
  constexpr int LOADS = (BM * BK) / 256;
  T pa[LOADS], pb[LOADS];
  auto gather = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      // consecutive threads take consecutive k of one row: the canonical
      // index m*K + k keeps its low (k) bits within a warp's 16-lane runs
      const int i = tid + 256 * r;
      const int mm = i / BK, kk = i % BK;
      const int64_t m = m0 + mm, n = n0 + mm, k = k0 + kk;
      pa[r].x = 0; pa[r].y = 0;
      pb[r].x = 0; pb[r].y = 0;
      if (m < M && k < K) pa[r] = A[lut_map(la, (uint32_t)(m * K + k))];
      if (n < N && k < K) pb[r] = B[lut_map(lb, (uint32_t)(n * K + k))];
    }
  };
  gather(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + 256 * r;
      As[i % BK][i / BK] = pa[r];
      Bs[i % BK][i / BK] = pb[r];
    }
    __syncthreads();
    if (k0 + BK < K) gather(k0 + BK);
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc_re[i][j] += av[i].x * bv[j].x - av[i].y * bv[j].y;
          acc_im[i][j] += av[i].x * bv[j].y + av[i].y * bv[j].x;
        }
    }
    __syncthreads();
  }
  float vmax = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        T v; v.x = acc_re[i][j]; v.y = acc_im[i][j];
        C[m * N + n] = v;
        vmax = fmaxf(vmax, (float)fmax(fabs(v.x), fabs(v.y)));
      }
    }
  if (max_out) block_max_atomic(vmax, max_out);
}

// fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) variant of the wide tile for
// complex128 steps: same 64x64 output tile, K blocks of 16 gathered through
// the LUTs into planar (re | im) shared-memory tiles, 8 warps of 32x16
// outputs, four real products per complex fragment (re += ar br - ai bi,
// im += ar bi + ai br).  Exact IEEE fp64 products and sums, like the FMA path.
#ifndef TNB_DMMA_BLOCKS
#define TNB_DMMA_BLOCKS 1
#endif
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, TNB_DMMA_BLOCKS)
contract_dmma_kernel(const double2* __restrict__ A, const double2* __restrict__ B,
                     double2* __restrict__ C, int64_t M, int64_t N, int64_t K,
                     const ByteLut* __restrict__ gla, const ByteLut* __restrict__ glb,
                     unsigned int* __restrict__ max_out) {
  constexpr int BM = 64, BN = 64, BK = 16, PAD = 8, LD = BM + PAD;
  __shared__ uint32_t la[4][256];
  __shared__ uint32_t lb[4][256];
  __shared__ double As[2][BK][LD];  // [re|im][k][m]
  __shared__ double Bs[2][BK][LD];  // [re|im][k][n]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += 256) {
    la[i >> 8][i & 255] = gla->t[i >> 8][i & 255];
    lb[i >> 8][i & 255] = glb->t[i >> 8][i & 255];
  }
  const int64_t nbn = (N + BN - 1) / BN;
  const int64_t m0 = ((int64_t)blockIdx.x / nbn) * BM, n0 = ((int64_t)blockIdx.x % nbn) * BN;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;  // warp tile origin
  double acc[4][2][2][2];  // [m frag][n frag][re|im][2 values]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc[i][j][c][0] = acc[i][j][c][1] = 0.0;
  __syncthreads();
  constexpr int LOADS = (BM * BK) / 256;
  double2 pa[LOADS], pb[LOADS];
  auto gather = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + 256 * r;
      const int mm = i / BK, kk = i % BK;
      const int64_t m = m0 + mm, n = n0 + mm, k = k0 + kk;
      pa[r] = make_double2(0.0, 0.0);
      pb[r] = make_double2(0.0, 0.0);
      if (m < M && k < K) pa[r] = A[lut_map(la, (uint32_t)(m * K + k))];
      if (n < N && k < K) pb[r] = B[lut_map(lb, (uint32_t)(n * K + k))];
    }
  };
  gather(0);
  const int fr = lane >> 2, fk = lane & 3;  // fragment row/col and k
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + 256 * r;
      const int mm = i / BK, kk = i % BK;
      As[0][kk][mm] = pa[r].x;
      As[1][kk][mm] = pa[r].y;
      Bs[0][kk][mm] = pb[r].x;
      Bs[1][kk][mm] = pb[r].y;
    }
    __syncthreads();
    if (k0 + BK < K) gather(k0 + BK);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[4], ai[4], br[2], bi[2], bn[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ar[i] = As[0][k4 + fk][wm + 8 * i + fr];
        ai[i] = As[1][k4 + fk][wm + 8 * i + fr];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        br[j] = Bs[0][k4 + fk][wn + 8 * j + fr];
        bi[j] = Bs[1][k4 + fk][wn + 8 * j + fr];
        bn[j] = -bi[j];
      }
      // two passes over the 16 accumulators so that the two products into
      // one accumulator are 16 DMMAs apart (back to back they stall on the
      // DMMA latency: "wait" was 30 % of the issue gaps)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma_8x8x4(acc[i][j][0], ar[i], br[j]);
          dmma_8x8x4(acc[i][j][1], ar[i], bi[j]);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma_8x8x4(acc[i][j][0], ai[i], bn[j]);
          dmma_8x8x4(acc[i][j][1], ai[i], br[j]);
        }
    }
    __syncthreads();
  }
  float vmax = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t m = m0 + wm + 8 * i + fr, n = n0 + wn + 8 * j + 2 * fk + e;
        if (m < M && n < N) {
          const double2 v = make_double2(acc[i][j][0][e], acc[i][j][1][e]);
          C[m * N + n] = v;
          vmax = fmaxf(vmax, (float)fmax(fabs(v.x), fabs(v.y)));
        }
      }
  if (max_out) block_max_atomic(vmax, max_out);
}

template <typename T>
__global__ void __launch_bounds__(256)
contract_simt_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                     int64_t M, int64_t N, int64_t K, const ByteLut* __restrict__ gla,
                     const ByteLut* __restrict__ glb, unsigned int* __restrict__ max_out) {
  simt_tile<T>(A, B, C, M, N, K, gla, glb, max_out, blockIdx.x);
}

// Several independent small SIMT steps in one launch (one block per 32x32
// tile of any of them): removes the per-step launch latency that dominates
// the ~160 tiny contraction steps of a slice.
template <typename T>
__global__ void __launch_bounds__(256)
contract_simt_batch_kernel(const SimtStepDesc* __restrict__ d, int n) {
  int lo = 0, hi = n;  // last descriptor with block0 <= blockIdx.x
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (d[mid].block0 <= (int64_t)blockIdx.x) lo = mid; else hi = mid;
  }
  const SimtStepDesc& s = d[lo];
  simt_tile<T>((const T*)s.A, (const T*)s.B, (T*)s.C, s.M, s.N, s.K, s.lut_a, s.lut_b, s.max_out,
               (int64_t)blockIdx.x - s.block0);
}

// ---------------------------------------------------------------------------
// Small-K contraction (outer-product-like steps, K <= 8, big outputs): each
// thread produces 4 consecutive output columns of one row with two 16-byte
// (float2) or four 16-byte (double2) stores, so the kernel runs at HBM write
// speed instead of the 32x32-tile kernel's padded K loop.
__device__ __forceinline__ void split2(float a, float b, __half2& hi, __half2& lo);

// fused output of the small-K kernel: C[m][n0..n0+3] as the tensor-core
// consumer's staged operand (see FuseOut / gemm_tc.cu fused_store)
__device__ __forceinline__ void smallk_fused_store(const FuseOut& fo, const uint32_t (*fm)[256],
                                                   const uint32_t (*fn)[256], int64_t m, int64_t n0,
                                                   const float* re, const float* im, float so) {
  const uint32_t base = lut_map(fm, (uint32_t)m) | lut_map(fn, (uint32_t)n0);
  if (fo.vec) {  // n bits 0,1 are destination bits 0,1: 16-B stores
    if (fo.mode == 1) {
      __half2 h[4], o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) split2(re[j] * so, im[j] * so, h[j], o[j]);
      *reinterpret_cast<uint4*>(fo.hi + base) = *reinterpret_cast<const uint4*>(h);
      *reinterpret_cast<uint4*>(fo.lo + base) = *reinterpret_cast<const uint4*>(o);
    } else {
      __half2 h0[4], o0[4], h1[4], o1[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        split2(re[j] * so, -im[j] * so, h0[j], o0[j]);
        split2(im[j] * so, re[j] * so, h1[j], o1[j]);
      }
      const uint32_t b1 = base + (1u << fo.L);
      *reinterpret_cast<uint4*>(fo.hi + base) = *reinterpret_cast<const uint4*>(h0);
      *reinterpret_cast<uint4*>(fo.lo + base) = *reinterpret_cast<const uint4*>(o0);
      *reinterpret_cast<uint4*>(fo.hi + b1) = *reinterpret_cast<const uint4*>(h1);
      *reinterpret_cast<uint4*>(fo.lo + b1) = *reinterpret_cast<const uint4*>(o1);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = base | fo.dlow[j];
    if (fo.mode == 1) {
      __half2 h, o;
      split2(re[j] * so, im[j] * so, h, o);
      fo.hi[a] = h;
      fo.lo[a] = o;
    } else {
      __half2 h0, o0, h1, o1;
      split2(re[j] * so, -im[j] * so, h0, o0);
      split2(im[j] * so, re[j] * so, h1, o1);
      const uint32_t a1 = a + (1u << fo.L);
      fo.hi[a] = h0; fo.lo[a] = o0;
      fo.hi[a1] = h1; fo.lo[a1] = o1;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
contract_smallk_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                       int64_t M, int64_t N, int K, const ByteLut* __restrict__ gla,
                       const ByteLut* __restrict__ glb, const ByteLut* __restrict__ gle,
                       unsigned int* __restrict__ max_out, const __grid_constant__ FuseOut fo) {
  using S = typename Scalar<T>::type;
  if (fo.redo && !fused_redo_fires(fo)) return;  // scale-guard re-run (FuseOut::redo)
  __shared__ uint32_t la[4][256];
  __shared__ uint32_t lb[4][256];
  __shared__ uint32_t fm[4][256];
  __shared__ uint32_t fn[4][256];
  __shared__ uint32_t le[4][256];
  const bool fused = std::is_same<T, float2>::value && fo.mode != 0;
  for (int i = threadIdx.x; i < 1024; i += 256) {
    la[i >> 8][i & 255] = gla->t[i >> 8][i & 255];
    lb[i >> 8][i & 255] = glb->t[i >> 8][i & 255];
    if (gle) le[i >> 8][i & 255] = gle->t[i >> 8][i & 255];
    if (fused) {
      fm[i >> 8][i & 255] = fo.lut_m->t[i >> 8][i & 255];
      fn[i >> 8][i & 255] = fo.lut_n->t[i >> 8][i & 255];
    }
  }
  const float so = fused ? scale_from_src(fo.scale) : 1.f;
  __syncthreads();
  const int64_t nq = N >> 2;
  const int64_t total = M * nq;
  float vmax = 0.f;
  for (int64_t idx = (int64_t)blockIdx.x * 256 + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * 256) {
    // thread-quad index -> output quad: the enumeration LUT keeps the 5 lane
    // bits on the output's lowest quad bits (coalesced stores) and puts the
    // big operand's lowest storage bits right above them, so the lines a
    // warp gathers are consumed by neighbouring warps while still in L2
    const int64_t cq = gle ? (int64_t)lut_map(le, (uint32_t)idx) : idx;
    const int64_t m = cq / nq, n0 = (cq - m * nq) << 2;
    S re[4] = {0, 0, 0, 0}, im[4] = {0, 0, 0, 0};
    // K is a power of two <= 8 and n0 a multiple of 4, so the canonical
    // indices m*K + k and (n0 + j)*K + k split into disjoint bit fields: one
    // full LUT lookup per row / column, then a byte-table OR per (j, k)
    const uint32_t abase = lut_map(la, (uint32_t)(m * K));
    const uint32_t bbase = lut_map(lb, (uint32_t)(n0 * K));
    for (int k = 0; k < K; ++k) {
      const T a = A[abase | la[0][k]];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const T b = B[bbase | lb[0][j * K + k]];
        re[j] += a.x * b.x - a.y * b.y;
        im[j] += a.x * b.y + a.y * b.x;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) vmax = fmaxf(vmax, (float)fmax(fabs(re[j]), fabs(im[j])));
    if constexpr (std::is_same<T, float2>::value) {
      if (fused) {
        smallk_fused_store(fo, fm, fn, m, n0, re, im, so);
        continue;
      }
    }
    T* dst = C + m * N + n0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      T v; v.x = re[j]; v.y = im[j];
      dst[j] = v;
    }
  }
  if (max_out) block_max_atomic(vmax, max_out);
}

// ---------------------------------------------------------------------------
// K4: bit permutation out[j] = in[lut(j)].
template <typename T>
__global__ void permute_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t elems,
                               const ByteLut* __restrict__ glut) {
  __shared__ uint32_t l[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) l[i >> 8][i & 255] = glut->t[i >> 8][i & 255];
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = in[lut_map(l, (uint32_t)j)];
}

// ---------------------------------------------------------------------------
// K5: binary-counter merge of `_fixed_tree_sum`: v = x; v = s_i + v for the
// n_merge occupied levels (oldest first), stored at dst.  Same IEEE ops as
// the reference's `x = prev + x` chain.
template <typename T>
__global__ void counter_merge_kernel(const T* __restrict__ x, const T* slots, int64_t stride,
                                     int n_merge, T* dst, int64_t elems) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x) {
    T v = x[j];
    for (int i = 0; i < n_merge; ++i) v = cadd(slots[(size_t)i * stride + j], v);
    dst[j] = v;
  }
}

template <typename T>
__global__ void add_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                           int64_t elems) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = cadd(a[j], b[j]);
}

template <typename T>
__global__ void copy_kernel(const T* __restrict__ a, T* __restrict__ out, int64_t elems) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = a[j];
}

// ---------------------------------------------------------------------------
// Tensor-core operand staging.  Power-of-two scaling keeps the fp16 split
// exact in range: max|x| * s lands in [2^14, 2^15); hi = fp16(x s),
// lo = fp16(x s - hi).  Unscaling by 1/(sA sB) is exact.
__device__ __forceinline__ float scale_from_bits(unsigned int bits) {
  const float m = __uint_as_float(bits);
  if (!(m > 0.f)) return 1.f;
  int e;
  frexpf(m, &e);  // m = f * 2^e, f in [0.5, 1)
  int p = 15 - e;
  p = p > 126 ? 126 : (p < -126 ? -126 : p);
  return ldexpf(1.f, p);
}

__global__ void absmax_kernel(const float2* __restrict__ A, int64_t n, unsigned int* __restrict__ maxbits) {
  float m = 0.f;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = A[j];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  block_max_atomic(m, maxbits);
}

__device__ __forceinline__ void split2(float a, float b, __half2& hi, __half2& lo) {
  hi = __floats2half2_rn(a, b);
  const float2 h = __half22float2(hi);
  lo = __floats2half2_rn(a - h.x, b - h.y);
}

// Tiled permute + fp16 split (+ 2x2 real expansion for the cols operand).
// A tile is the set of canonical indices spanned by the low destination
// bits and the canonical bits that land on the low source bits: it is read
// in source order (coalesced 256-B runs) into shared memory and written in
// destination order (coalesced runs).  rows: hi/lo[j] for j = r*K + k;
// cols (expand): rows 2n / 2n+1 of the 2x2 real representation.
template <bool kExpand, int EPT>
__global__ void __launch_bounds__(256)
stage_kernel(const float2* __restrict__ src, StageTables tb, int64_t K, int logK,
             const unsigned int* __restrict__ maxbits, __half2* __restrict__ hi,
             __half2* __restrict__ lo) {
  extern __shared__ float2 tile[];  // padded by one element per 32
  __shared__ uint32_t ls[4][256];
  __shared__ uint32_t ld[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    ls[i >> 8][i & 255] = tb.tile_src->t[i >> 8][i & 255];
    ld[i >> 8][i & 255] = tb.tile_dst->t[i >> 8][i & 255];
  }
  const int tsize = 1 << tb.nU;
  const float s = scale_from_bits(*maxbits);
  __syncthreads();
  for (int64_t T = blockIdx.x; T < tb.n_tiles; T += gridDim.x) {
    const uint32_t sbase = lut_map(ls, (uint32_t)T);
    const uint32_t dbase = lut_map(ld, (uint32_t)T);
    // read phase: EPT independent loads in flight per thread (source order)
    float2 v[EPT];
    uint32_t tt[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int i = threadIdx.x + 256 * j;
      if (i < tsize) {
        tt[j] = __ldg(tb.rd_t + i);
        v[j] = src[sbase + __ldg(tb.rd_src + i)];
      }
    }
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int i = threadIdx.x + 256 * j;
      if (i < tsize) tile[tt[j] + (tt[j] >> 5)] = v[j];
    }
    __syncthreads();
    // write phase: destination order
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int t = threadIdx.x + 256 * j;
      if (t >= tsize) break;
      const float2 x = tile[t + (t >> 5)];
      const uint32_t d = dbase + __ldg(tb.t_dst + t);
      if (!kExpand) {
        __half2 h, o;
        split2(x.x * s, x.y * s, h, o);
        hi[d] = h;
        lo[d] = o;
      } else {
        // d = (k_hi, n, k_lo) with 2^logK = k_lo extent: rows 2n / 2n+1 of
        // the block are 2^logK apart
        const uint64_t r0 = (uint64_t)d + (((uint64_t)d >> logK) << logK);
        const uint64_t r1 = r0 + (1ull << logK);
        __half2 h0, o0, h1, o1;
        split2(x.x * s, -x.y * s, h0, o0);
        split2(x.y * s, x.x * s, h1, o1);
        hi[r0] = h0; lo[r0] = o0;
        hi[r1] = h1; lo[r1] = o1;
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Same tiles as stage_kernel (tile = 2^nU >= 1024 elements here), with
//  * the gather of tile T+1 (cp.async, source order, into the second shared
//    buffer) in flight while tile T is split and written, so the HBM reads
//    no longer wait behind each tile's write phase;
//  * all per-element tables in registers (a thread's slots are the same in
//    every tile);
//  * 4 consecutive tile elements per thread in the write phase: the low 5
//    tile bits are the low 5 destination bits, so they land on 4 contiguous
//    destination slots (16-B stores).
// Shared layout: 2 pad elements per 32 keep each 4-group 16-B aligned.
constexpr int kAsyncPad = 2;
template <bool kExpand, int EPT>
__global__ void __launch_bounds__(256)
stage_async_kernel(const float2* __restrict__ src, StageTables tb, int logK,
                   const unsigned int* __restrict__ maxbits, __half2* __restrict__ hi,
                   __half2* __restrict__ lo) {
  static_assert(EPT % 4 == 0, "4 elements per write group");
  constexpr int G = EPT / 4;  // write groups per thread
  extern __shared__ float4 tile4[];  // two padded buffers (float2 units below)
  float2* tile = reinterpret_cast<float2*>(tile4);
  __shared__ uint32_t ls[4][256];
  __shared__ uint32_t ld[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    ls[i >> 8][i & 255] = tb.tile_src->t[i >> 8][i & 255];
    ld[i >> 8][i & 255] = tb.tile_dst->t[i >> 8][i & 255];
  }
  const int tsize = 1 << tb.nU;  // == 256 * EPT
  const int bstride = tsize + kAsyncPad * (tsize >> 5);
  uint32_t tt[EPT], so[EPT], dq[G];
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int i = threadIdx.x + 256 * j;
    const uint32_t t = __ldg(tb.rd_t + i);
    tt[j] = t + kAsyncPad * (t >> 5);
    so[j] = __ldg(tb.rd_src + i);
  }
#pragma unroll
  for (int g = 0; g < G; ++g) dq[g] = __ldg(tb.t_dst + 4 * (threadIdx.x + 256 * g));
  const float s = scale_from_bits(*maxbits);
  __syncthreads();
  auto gather = [&](int64_t T, int buf) {
    const float2* sb = src + lut_map(ls, (uint32_t)T);
    float2* tb_ = tile + buf * bstride;
#pragma unroll
    for (int j = 0; j < EPT; ++j) cp_async8(tb_ + tt[j], sb + so[j]);
  };
  int buf = 0;
  if ((int64_t)blockIdx.x < tb.n_tiles) gather(blockIdx.x, 0);
  cp_async_commit();
  for (int64_t T = blockIdx.x; T < tb.n_tiles; T += gridDim.x, buf ^= 1) {
    const int64_t Tn = T + gridDim.x;
    if (Tn < tb.n_tiles) gather(Tn, buf ^ 1);
    cp_async_commit();
    cp_async_wait1();  // this thread's copies of tile T have landed
    __syncthreads();   // ... and everyone else's
    const float2* tl = tile + buf * bstride;
    const uint32_t dbase = lut_map(ld, (uint32_t)T);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int t0 = 4 * (threadIdx.x + 256 * g);
      const float4* p = reinterpret_cast<const float4*>(tl + t0 + kAsyncPad * (t0 >> 5));
      const float4 x01 = p[0], x23 = p[1];
      const float re[4] = {x01.x, x01.z, x23.x, x23.z};
      const float im[4] = {x01.y, x01.w, x23.y, x23.w};
      const uint32_t d = dbase + dq[g];
      if (!kExpand) {
        __half2 h[4], o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split2(re[e] * s, im[e] * s, h[e], o[e]);
        *reinterpret_cast<uint4*>(hi + d) = *reinterpret_cast<const uint4*>(h);
        *reinterpret_cast<uint4*>(lo + d) = *reinterpret_cast<const uint4*>(o);
      } else {
        const uint64_t r0 = (uint64_t)d + (((uint64_t)d >> logK) << logK);
        const uint64_t r1 = r0 + (1ull << logK);
        __half2 h0[4], o0[4], h1[4], o1[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          split2(re[e] * s, -im[e] * s, h0[e], o0[e]);
          split2(im[e] * s, re[e] * s, h1[e], o1[e]);
        }
        *reinterpret_cast<uint4*>(hi + r0) = *reinterpret_cast<const uint4*>(h0);
        *reinterpret_cast<uint4*>(lo + r0) = *reinterpret_cast<const uint4*>(o0);
        *reinterpret_cast<uint4*>(hi + r1) = *reinterpret_cast<const uint4*>(h1);
        *reinterpret_cast<uint4*>(lo + r1) = *reinterpret_cast<const uint4*>(o1);
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's gather
  }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t elems,
                                     float* __restrict__ C, const ScaleSrc scale_rows,
                                     const ScaleSrc scale_cols, unsigned int* __restrict__ max_out) {
  const float alpha = 1.f / (scale_from_src(scale_rows) * scale_from_src(scale_cols));
  float m = 0.f;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[(int64_t)s * elems + j];
    acc *= alpha;
    C[j] = acc;
    m = fmaxf(m, fabsf(acc));
  }
  if (max_out) block_max_atomic(m, max_out);
}

inline int grid_for(int64_t elems, int threads) {
  int64_t g = (elems + threads - 1) / threads;
  const int64_t cap = (int64_t)kSms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

void build_lut(const std::vector<int>& src_bit, ByteLut* out) {
  if (src_bit.size() > 32) throw Error(TNB_ERR_SHAPE, "tensor rank above 32 is not supported");
  for (int t = 0; t < 4; ++t)
    for (int v = 0; v < 256; ++v) {
      uint32_t o = 0;
      for (int i = 0; i < 8; ++i) {
        const int p = 8 * t + i;
        if (((v >> i) & 1) && p < (int)src_bit.size()) o |= (1u << src_bit[p]);
      }
      out->t[t][v] = o;
    }
}

template <typename T>
void launch_prepare_leaves(const T* leaf_pool, T* slice_pool, const SlicedLeafDesc* descs,
                           int n_descs, const uint32_t* keep_tables, uint64_t mask, cudaStream_t s) {
  if (n_descs == 0) return;
  prepare_leaves_kernel<T><<<n_descs, 64, 0, s>>>(leaf_pool, slice_pool, descs, keep_tables, mask);
  check_launch("prepare_leaves");
}

template <typename T>
void launch_contract_simt(const T* A, const T* B, T* C, int64_t M, int64_t N, int64_t K,
                          const ByteLut* lutA, const ByteLut* lutB, const ByteLut* lutE,
                          unsigned int* max_out, const FuseOut* fuse, cudaStream_t s) {
  if (simt_uses_smallk(M, N, K)) {
    // outer-product-like: stream the output
    const FuseOut fo = fuse ? *fuse : FuseOut{};
    // resident blocks per SM: fewer keeps the gathered lines in flight
    // inside L2 (the operand gathers are scattered below the 2^11-quad window)
    static const int per_sm = [] { const char* e = getenv("TNB_SMALLK_BLOCKS"); return e ? atoi(e) : 16; }();
    int64_t g = grid_for(M * (N >> 2), 256);
    if (g > (int64_t)kSms * per_sm) g = (int64_t)kSms * per_sm;
    contract_smallk_kernel<T><<<(int)g, 256, 0, s>>>(A, B, C, M, N, (int)K, lutA,
                                                                            lutB, lutE, max_out, fo);
    check_launch("contract_smallk");
    return;
  }
  if (fuse && fuse->mode != 0) throw Error(TNB_ERR_SHAPE, "fused output planned for a tiled SIMT step");
  if (simt_uses_wide(M, N, K)) {
    const int64_t wb = ((M + 63) / 64) * ((N + 63) / 64);
    if (wb > 0x7fffffffll) throw Error(TNB_ERR_SHAPE, "SIMT contraction too large");
    static const int dmma = [] { const char* e = getenv("TNB_DMMA"); return e ? atoi(e) : 1; }();
    if constexpr (std::is_same<T, double2>::value) {
      if (dmma) {
        contract_dmma_kernel<<<(unsigned)wb, 256, 0, s>>>(A, B, C, M, N, K, lutA, lutB, max_out);
        check_launch("contract_dmma");
        return;
      }
    }
    contract_wide_kernel<T><<<(unsigned)wb, 256, 0, s>>>(A, B, C, M, N, K, lutA, lutB, max_out);
    check_launch("contract_wide");
    return;
  }
  const int64_t blocks = ((M + 31) / 32) * ((N + 31) / 32);
  if (blocks > 0x7fffffffll) throw Error(TNB_ERR_SHAPE, "SIMT contraction too large");
  contract_simt_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(A, B, C, M, N, K, lutA, lutB, max_out);
  check_launch("contract_simt");
}

int64_t simt_tiles(int64_t M, int64_t N) { return ((M + 31) / 32) * ((N + 31) / 32); }

template <typename T>
void launch_contract_simt_batch(const SimtStepDesc* descs, int n, int64_t blocks, cudaStream_t s) {
  if (blocks > 0x7fffffffll) throw Error(TNB_ERR_SHAPE, "SIMT batch too large");
  contract_simt_batch_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(descs, n);
  check_launch("contract_simt_batch");
}

template <typename T>
void launch_permute(const T* in, T* out, int64_t elems, const ByteLut* lut, cudaStream_t s) {
  permute_kernel<T><<<grid_for(elems, 256), 256, 0, s>>>(in, out, elems, lut);
  check_launch("permute");
}

template <typename T>
void launch_counter_merge(const T* x, const T* slots, int64_t stride, int n_merge, T* dst,
                          int64_t elems, cudaStream_t s) {
  counter_merge_kernel<T><<<grid_for(elems, 256), 256, 0, s>>>(x, slots, stride, n_merge, dst, elems);
  check_launch("counter_merge");
}

template <typename T>
void launch_add(const T* a, const T* b, T* out, int64_t elems, cudaStream_t s) {
  add_kernel<T><<<grid_for(elems, 256), 256, 0, s>>>(a, b, out, elems);
  check_launch("add");
}

template <typename T>
void launch_copy(const T* a, T* out, int64_t elems, cudaStream_t s) {
  copy_kernel<T><<<grid_for(elems, 256), 256, 0, s>>>(a, out, elems);
  check_launch("copy");
}

void launch_absmax(const float2* A, int64_t n, unsigned int* maxbits, cudaStream_t s) {
  TNB_CUDA(cudaMemsetAsync(maxbits, 0, sizeof(unsigned int), s));
  absmax_kernel<<<grid_for(n, 512), 512, 0, s>>>(A, n, maxbits);
  check_launch("absmax");
}

void build_stage_tables(const std::vector<int>& canon_rowmajor, int64_t K, StageHost* out) {
  const int r = (int)canon_rowmajor.size();
  // destination bit order of the K-blocked layout: k_lo, row bits, k_hi
  int logK = 0;
  while ((1ll << logK) < K) ++logK;
  std::vector<int> canon_to_src;
  if (logK > kKBlockLog) {
    for (int p = 0; p < kKBlockLog; ++p) canon_to_src.push_back(canon_rowmajor[p]);
    for (int p = logK; p < r; ++p) canon_to_src.push_back(canon_rowmajor[p]);
    for (int p = kKBlockLog; p < logK; ++p) canon_to_src.push_back(canon_rowmajor[p]);
  } else {
    canon_to_src = canon_rowmajor;
  }
  const int Ld = std::min(stage_run_bits(), r), Ls = std::min(stage_run_bits(), r);
  std::vector<int> src_to_canon(r, -1);
  for (int p = 0; p < r; ++p) src_to_canon[canon_to_src[p]] = p;
  std::vector<char> inU(r, 0);
  for (int p = 0; p < Ld; ++p) inU[p] = 1;
  for (int q = 0; q < Ls; ++q) inU[src_to_canon[q]] = 1;
  // grow the tile to 2^11 elements (or the whole tensor) with the next
  // lowest canonical bits so every tile keeps 256 threads busy
  {
    int cnt = 0;
    for (int p = 0; p < r; ++p) cnt += inU[p];
    for (int p = 0; p < r && cnt < std::min(r, stage_tile_bits()); ++p)
      if (!inU[p]) { inU[p] = 1; ++cnt; }
  }
  std::vector<int> U, V;
  for (int p = 0; p < r; ++p) (inU[p] ? U : V).push_back(p);
  std::vector<int> upos(r, -1);
  for (int u = 0; u < (int)U.size(); ++u) upos[U[u]] = u;
  // read order: source bits 0..Ls-1 fastest, then the remaining tile bits
  std::vector<int> read_map;
  std::vector<char> used(U.size(), 0);
  for (int q = 0; q < Ls; ++q) { read_map.push_back(upos[src_to_canon[q]]); used[upos[src_to_canon[q]]] = 1; }
  for (int u = 0; u < (int)U.size(); ++u) if (!used[u]) read_map.push_back(u);
  const int nU = (int)U.size();
  out->nU = nU;
  out->n_tiles = (int64_t)1 << (r - nU);
  out->rd_t.assign((size_t)1 << nU, 0);
  out->rd_src.assign((size_t)1 << nU, 0);
  out->t_dst.assign((size_t)1 << nU, 0);
  for (uint32_t i = 0; i < (1u << nU); ++i) {
    uint32_t t = 0, so = 0;
    for (int b = 0; b < nU; ++b)
      if ((i >> b) & 1) { t |= 1u << read_map[b]; so |= 1u << canon_to_src[U[read_map[b]]]; }
    out->rd_t[i] = t;
    out->rd_src[i] = so;
  }
  for (uint32_t t = 0; t < (1u << nU); ++t) {
    uint32_t d = 0;
    for (int u = 0; u < nU; ++u) if ((t >> u) & 1) d |= 1u << U[u];
    out->t_dst[t] = d;
  }
  // tile-id bits in canonical (destination) order by default; TNB_STAGE_ORDER=1
  // orders them by source bit instead (measured: no difference at C4)
  static const int tile_order = [] { const char* e = getenv("TNB_STAGE_ORDER"); return e ? atoi(e) : 0; }();
  if (tile_order == 1)
    std::sort(V.begin(), V.end(), [&](int x, int y) { return canon_to_src[x] < canon_to_src[y]; });
  std::vector<int> vs, vd;
  for (int p : V) { vs.push_back(canon_to_src[p]); vd.push_back(p); }
  build_lut(vs, &out->tile_src);
  build_lut(vd, &out->tile_dst);
}

void launch_stage(const float2* src, const StageTables& tb, int64_t K, bool expand,
                  const unsigned int* maxbits, __half* hi, __half* lo, cudaStream_t s) {
  int logK = 0;
  while ((1ll << logK) < K) ++logK;
  if (logK > kKBlockLog) logK = kKBlockLog;  // row length of the K-blocked layout
  const size_t smem = ((size_t)1 << tb.nU) * 8 + (((size_t)1 << tb.nU) / 32 + 1) * 8;
  int64_t g = tb.n_tiles;
  const int64_t cap = (int64_t)kSms * 8;
  if (g > cap) g = cap;
  const int ept = (1 << tb.nU) <= 256 ? 1 : (1 << tb.nU) / 256;
  static const int async = [] { const char* e = getenv("TNB_STAGE_ASYNC"); return e ? atoi(e) : 1; }();
  auto go = [&](auto kexp, auto kept) {
    constexpr bool kE = decltype(kexp)::value;
    constexpr int kP = decltype(kept)::value;
    bool done = false;
    if constexpr (kP >= 4) {
      auto kern = stage_async_kernel<kE, kP>;
      const size_t tsz = (size_t)1 << tb.nU;
      const size_t smem2 = 2 * 8 * (tsz + kAsyncPad * (tsz >> 5));
      int per_sm = 0;
      if (async) {
        if (smem2 > 48 * 1024)
          TNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        TNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem2));
      }
      // persistent grid of resident blocks, each looping (and prefetching) over tiles
      const int64_t g2 = (int64_t)kSms * per_sm;
      if (per_sm > 0 && tb.n_tiles > 2 * g2 && tsz == (size_t)256 * kP) {
        kern<<<(unsigned)g2, 256, smem2, s>>>(src, tb, logK, maxbits, reinterpret_cast<__half2*>(hi),
                                             reinterpret_cast<__half2*>(lo));
        done = true;
      }
    }
    if (!done) {
      stage_kernel<kE, kP><<<(unsigned)g, 256, smem, s>>>(
          src, tb, K, logK, maxbits, reinterpret_cast<__half2*>(hi), reinterpret_cast<__half2*>(lo));
    }
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  switch (ept) {
    case 1: expand ? go(T_{}, std::integral_constant<int, 1>{}) : go(F_{}, std::integral_constant<int, 1>{}); break;
    case 2: expand ? go(T_{}, std::integral_constant<int, 2>{}) : go(F_{}, std::integral_constant<int, 2>{}); break;
    case 4: expand ? go(T_{}, std::integral_constant<int, 4>{}) : go(F_{}, std::integral_constant<int, 4>{}); break;
    case 8: expand ? go(T_{}, std::integral_constant<int, 8>{}) : go(F_{}, std::integral_constant<int, 8>{}); break;
    default: expand ? go(T_{}, std::integral_constant<int, 16>{}) : go(F_{}, std::integral_constant<int, 16>{}); break;
  }
  check_launch("stage");
}

void launch_splitk_reduce(const float* ws, int splits, int64_t elems, float* C,
                          const ScaleSrc& scale_rows, const ScaleSrc& scale_cols,
                          unsigned int* max_out, cudaStream_t s) {
  splitk_reduce_kernel<<<grid_for(elems, 256), 256, 0, s>>>(ws, splits, elems, C, scale_rows,
                                                            scale_cols, max_out);
  check_launch("splitk_reduce");
}

#define TNB_INST(T)                                                                        \
  template void launch_prepare_leaves<T>(const T*, T*, const SlicedLeafDesc*, int,         \
                                         const uint32_t*, uint64_t, cudaStream_t);         \
  template void launch_contract_simt<T>(const T*, const T*, T*, int64_t, int64_t, int64_t, \
                                        const ByteLut*, const ByteLut*, const ByteLut*,    \
                                        unsigned int*, const FuseOut*, cudaStream_t);      \
  template void launch_contract_simt_batch<T>(const SimtStepDesc*, int, int64_t, cudaStream_t); \
  template void launch_permute<T>(const T*, T*, int64_t, const ByteLut*, cudaStream_t);    \
  template void launch_counter_merge<T>(const T*, const T*, int64_t, int, T*, int64_t, cudaStream_t); \
  template void launch_add<T>(const T*, const T*, T*, int64_t, cudaStream_t);              \
  template void launch_copy<T>(const T*, T*, int64_t, cudaStream_t);
TNB_INST(float2)
TNB_INST(double2)
#undef TNB_INST

}  // namespace tnb
