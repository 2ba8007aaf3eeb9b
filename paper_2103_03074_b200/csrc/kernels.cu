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

namespace tnb {

namespace {

constexpr int kSms = 148;

__device__ __forceinline__ uint32_t lut_map(const uint32_t (*t)[256], uint32_t j) {
  return t[0][j & 255u] | t[1][(j >> 8) & 255u] | t[2][(j >> 16) & 255u] | t[3][j >> 24];
}

template <typename T> struct Scalar;
template <> struct Scalar<float2> { using type = float; };
template <> struct Scalar<double2> { using type = double; };

template <typename T>
__device__ __forceinline__ T cadd(T a, T b) { T r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }

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
template <typename T>
__global__ void __launch_bounds__(256)
contract_simt_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                     int64_t M, int64_t N, int64_t K, const ByteLut* __restrict__ gla,
                     const ByteLut* __restrict__ glb) {
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
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
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
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        T v; v.x = acc_re[i][j]; v.y = acc_im[i][j];
        C[m * N + n] = v;
      }
    }
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

__global__ void absmax2_kernel(const float2* __restrict__ A, int64_t nA,
                               const float2* __restrict__ B, int64_t nB,
                               unsigned int* __restrict__ maxbits) {
  const float2* src = blockIdx.y == 0 ? A : B;
  const int64_t n = blockIdx.y == 0 ? nA : nB;
  float m = 0.f;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = src[j];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(&maxbits[blockIdx.y], __float_as_uint(m));
  }
}

__device__ __forceinline__ void split2(float a, float b, __half2& hi, __half2& lo) {
  hi = __floats2half2_rn(a, b);
  const float2 h = __half22float2(hi);
  lo = __floats2half2_rn(a - h.x, b - h.y);
}

// rows operand: hi/lo[m][2k + c] (K-major, Kp = 2K)
__global__ void split_rows_kernel(const float2* __restrict__ src, const ByteLut* __restrict__ glut,
                                  int64_t M, int64_t K, const unsigned int* __restrict__ maxbits,
                                  __half2* __restrict__ hi, __half2* __restrict__ lo) {
  __shared__ uint32_t l[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) l[i >> 8][i & 255] = glut->t[i >> 8][i & 255];
  __syncthreads();
  const float s = scale_from_bits(maxbits[0]);
  const int64_t n = M * K;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = src[lut_map(l, (uint32_t)j)];
    __half2 h, o;
    split2(v.x * s, v.y * s, h, o);
    hi[j] = h;  // element j = m*K + k -> half2 at [m][2k..2k+1]
    lo[j] = o;
  }
}

// cols operand, expanded to the real 2x2 representation:
// row 2n: (br, -bi), row 2n+1: (bi, br) along k' = 2k, 2k+1.
__global__ void split_cols_expand_kernel(const float2* __restrict__ src,
                                         const ByteLut* __restrict__ glut, int64_t N, int64_t K,
                                         const unsigned int* __restrict__ maxbits,
                                         __half2* __restrict__ hi, __half2* __restrict__ lo) {
  __shared__ uint32_t l[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) l[i >> 8][i & 255] = glut->t[i >> 8][i & 255];
  __syncthreads();
  const float s = scale_from_bits(maxbits[1]);
  const int64_t n = N * K;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nn = j / K, k = j - nn * K;
    const float2 v = src[lut_map(l, (uint32_t)j)];
    __half2 h0, o0, h1, o1;
    split2(v.x * s, -v.y * s, h0, o0);
    split2(v.y * s, v.x * s, h1, o1);
    const int64_t r0 = (2 * nn) * K + k, r1 = (2 * nn + 1) * K + k;  // half2 units per row = K
    hi[r0] = h0; lo[r0] = o0;
    hi[r1] = h1; lo[r1] = o1;
  }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t elems,
                                     float* __restrict__ C, const unsigned int* __restrict__ maxbits) {
  const float alpha = 1.f / (scale_from_bits(maxbits[0]) * scale_from_bits(maxbits[1]));
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < elems;
       j += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[(int64_t)s * elems + j];
    C[j] = acc * alpha;
  }
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
                          const ByteLut* lutA, const ByteLut* lutB, cudaStream_t s) {
  dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
  if (grid.y > 65535) throw Error(TNB_ERR_SHAPE, "SIMT contraction: M too large");
  contract_simt_kernel<T><<<grid, 256, 0, s>>>(A, B, C, M, N, K, lutA, lutB);
  check_launch("contract_simt");
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

void launch_absmax2(const float2* A, int64_t nA, const float2* B, int64_t nB,
                    unsigned int* maxbits, cudaStream_t s) {
  TNB_CUDA(cudaMemsetAsync(maxbits, 0, 2 * sizeof(unsigned int), s));
  const int64_t n = nA > nB ? nA : nB;
  dim3 grid(grid_for(n, 512), 2);
  absmax2_kernel<<<grid, 512, 0, s>>>(A, nA, B, nB, maxbits);
  check_launch("absmax2");
}

void launch_split_rows(const float2* src, const ByteLut* lut, int64_t M, int64_t K,
                       const unsigned int* maxbits, __half* hi, __half* lo, cudaStream_t s) {
  split_rows_kernel<<<grid_for(M * K, 256), 256, 0, s>>>(src, lut, M, K, maxbits,
                                                          reinterpret_cast<__half2*>(hi),
                                                          reinterpret_cast<__half2*>(lo));
  check_launch("split_rows");
}

void launch_split_cols_expand(const float2* src, const ByteLut* lut, int64_t N, int64_t K,
                              const unsigned int* maxbits, __half* hi, __half* lo, cudaStream_t s) {
  split_cols_expand_kernel<<<grid_for(N * K, 256), 256, 0, s>>>(
      src, lut, N, K, maxbits, reinterpret_cast<__half2*>(hi), reinterpret_cast<__half2*>(lo));
  check_launch("split_cols_expand");
}

void launch_splitk_reduce(const float* ws, int splits, int64_t elems, float* C,
                          const unsigned int* maxbits, cudaStream_t s) {
  splitk_reduce_kernel<<<grid_for(elems, 256), 256, 0, s>>>(ws, splits, elems, C, maxbits);
  check_launch("splitk_reduce");
}

#define TNB_INST(T)                                                                        \
  template void launch_prepare_leaves<T>(const T*, T*, const SlicedLeafDesc*, int,         \
                                         const uint32_t*, uint64_t, cudaStream_t);         \
  template void launch_contract_simt<T>(const T*, const T*, T*, int64_t, int64_t, int64_t, \
                                        const ByteLut*, const ByteLut*, cudaStream_t);     \
  template void launch_permute<T>(const T*, T*, int64_t, const ByteLut*, cudaStream_t);    \
  template void launch_counter_merge<T>(const T*, const T*, int64_t, int, T*, int64_t, cudaStream_t); \
  template void launch_add<T>(const T*, const T*, T*, int64_t, cudaStream_t);              \
  template void launch_copy<T>(const T*, T*, int64_t, cudaStream_t);
TNB_INST(float2)
TNB_INST(double2)
#undef TNB_INST

}  // namespace tnb
