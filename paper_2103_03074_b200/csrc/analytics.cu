// On-device output-distribution analytics: the
// reductions behind tncut analytics.py (XEB :46-58, Porter-Thomas KS :70-79,
// histogram :90-121, post-selection curve :124-143, marginal/conditional
// :159-177) on a probability vector that already lives in HBM next to the
// amplitudes the tail produced.
//
// Determinism: sums use a fixed grid and a fixed per-block tree, so repeated
// calls return identical bits; min/max/histogram counts are exact.  Sorting
// (post-selection, KS) uses the toolkit's CUB radix sort on the fp64 bit
// patterns (p >= 0, so the unsigned order is the numeric order).
#include "tnb_internal.h"

#include <cub/cub.cuh>

#include <memory>

namespace tnb {
namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;  // 2 per SM, fixed: the summation tree must not depend on the device

template <typename T>
__global__ void probabilities_kernel(const T* __restrict__ a, int64_t n, double* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double re = (double)a[i].x, im = (double)a[i].y;
    p[i] = re * re + im * im;
  }
}

struct SumMinMax {
  double s, lo, hi, lo_pos;  // sum, min, max, min over p > 0
};

__device__ __forceinline__ SumMinMax smm_combine(SumMinMax a, SumMinMax b) {
  return {a.s + b.s, fmin(a.lo, b.lo), fmax(a.hi, b.hi), fmin(a.lo_pos, b.lo_pos)};
}

// per-block partial (sum, min, max) over a fixed contiguous chunk, tree order
__global__ void __launch_bounds__(kRedThreads)
reduce_partials_kernel(const double* __restrict__ p, int64_t n, SumMinMax* __restrict__ part) {
  __shared__ SumMinMax sh[kRedThreads];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  SumMinMax acc{0.0, INFINITY, -INFINITY, INFINITY};
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kRedThreads) {
    const double v = p[i];
    acc = smm_combine(acc, {v, v, v, v > 0.0 ? v : INFINITY});
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = smm_combine(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void reduce_final_kernel(const SumMinMax* __restrict__ part, int n, SumMinMax* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    SumMinMax acc{0.0, INFINITY, -INFINITY, INFINITY};
    for (int i = 0; i < n; ++i) acc = smm_combine(acc, part[i]);  // fixed left-to-right
    *out = acc;
  }
}

// np.histogram with explicit edges: bin i holds edges[i] <= x < edges[i+1],
// the last bin also x == edges[bins]; values outside are not counted
__global__ void histogram_kernel(const double* __restrict__ p, int64_t n, double scale,
                                 const double* __restrict__ edges, int bins,
                                 unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned long long local[];
  for (int i = threadIdx.x; i < bins; i += blockDim.x) local[i] = 0;
  __syncthreads();
  const double e0 = edges[0], eb = edges[bins];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = p[i] * scale;
    if (!(x >= e0 && x <= eb)) continue;
    int lo = 0, hi = bins;  // largest k with edges[k] <= x, clamped to bins-1
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (edges[mid] <= x) lo = mid; else hi = mid;
    }
    atomicAdd(&local[lo], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x)
    if (local[i]) atomicAdd(&counts[i], local[i]);
}

// any p[i+1] > p[i] (not sorted descending)
__global__ void check_desc_kernel(const double* __restrict__ p, int64_t n, int* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += (int64_t)gridDim.x * blockDim.x)
    if (p[i + 1] > p[i]) { atomicExch(bad, 1); return; }
}

// KS distance of x = scale * p (sorted ascending) against Exp(1):
// max_i max(|g_i - cdf_i|, |g_i - 1/L - cdf_i|), g_i = (i+1)/L
__global__ void ks_kernel(const double* __restrict__ p, int64_t n, double scale, unsigned long long* __restrict__ out) {
  double m = 0.0;
  const double L = (double)n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double cdf = 1.0 - exp(-p[i] * scale);
    const double g = (double)(i + 1) / L;
    m = fmax(m, fmax(fabs(g - cdf), fabs(g - 1.0 / L - cdf)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));  // m >= 0
}

__global__ void gather_kernel(const double* __restrict__ csum, const int64_t* __restrict__ ks, int nk,
                              double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nk) out[i] = csum[ks[i] - 1];
}

int grid_of(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8));
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { TNB_CUDA(cudaMalloc(&p, bytes ? bytes : 8)); }
  ~Dev() { if (p) cudaFree(p); }
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { TNB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() { if (s) cudaStreamDestroy(s); }
};

}  // namespace

void prob_from_amps(int precision, const void* amps, int64_t n, double* p) {
  Stream st;
  if (precision == TNB_SINGLE)
    probabilities_kernel<float2><<<grid_of(n), 256, 0, st.s>>>((const float2*)amps, n, p);
  else
    probabilities_kernel<double2><<<grid_of(n), 256, 0, st.s>>>((const double2*)amps, n, p);
  check_launch("probabilities");
  TNB_CUDA(cudaStreamSynchronize(st.s));
}

void prob_reduce(const double* p, int64_t n, double* out4) {
  Stream st;
  Dev part(kRedBlocks * sizeof(SumMinMax)), res(sizeof(SumMinMax));
  reduce_partials_kernel<<<kRedBlocks, kRedThreads, 0, st.s>>>(p, n, (SumMinMax*)part.p);
  reduce_final_kernel<<<1, 32, 0, st.s>>>((const SumMinMax*)part.p, kRedBlocks, (SumMinMax*)res.p);
  check_launch("prob_reduce");
  SumMinMax h;
  TNB_CUDA(cudaMemcpyAsync(&h, res.p, sizeof(h), cudaMemcpyDeviceToHost, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
  out4[0] = h.s;
  out4[1] = h.lo;
  out4[2] = h.hi;
  out4[3] = h.lo_pos;  // +inf when no p > 0
}

void prob_histogram(const double* p, int64_t n, double scale, const double* edges, int bins, int64_t* counts) {
  if (bins < 1) throw Error(TNB_ERR_ARG, "bins must be >= 1");
  Stream st;
  Dev de((bins + 1) * sizeof(double)), dc(bins * sizeof(unsigned long long));
  TNB_CUDA(cudaMemcpyAsync(de.p, edges, (bins + 1) * sizeof(double), cudaMemcpyHostToDevice, st.s));
  TNB_CUDA(cudaMemsetAsync(dc.p, 0, bins * sizeof(unsigned long long), st.s));
  const size_t smem = bins * sizeof(unsigned long long);
  if (smem > 48 * 1024) throw Error(TNB_ERR_ARG, "too many histogram bins");
  histogram_kernel<<<grid_of(n), 256, smem, st.s>>>(p, n, scale, (const double*)de.p, bins,
                                                   (unsigned long long*)dc.p);
  check_launch("histogram");
  TNB_CUDA(cudaMemcpyAsync(counts, dc.p, bins * sizeof(int64_t), cudaMemcpyDeviceToHost, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
}

void prob_sort(double* p, int64_t n, int descending) {
  if (n > (int64_t)INT32_MAX) throw Error(TNB_ERR_ARG, "sort size above 2^31");
  Stream st;
  Dev out(n * sizeof(double));
  auto* in_k = reinterpret_cast<unsigned long long*>(p);
  auto* out_k = reinterpret_cast<unsigned long long*>(out.p);
  size_t tmp = 0;
  if (descending)
    TNB_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp, in_k, out_k, (int)n, 0, 64, st.s));
  else
    TNB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in_k, out_k, (int)n, 0, 64, st.s));
  Dev work(tmp);
  if (descending)
    TNB_CUDA(cub::DeviceRadixSort::SortKeysDescending(work.p, tmp, in_k, out_k, (int)n, 0, 64, st.s));
  else
    TNB_CUDA(cub::DeviceRadixSort::SortKeys(work.p, tmp, in_k, out_k, (int)n, 0, 64, st.s));
  TNB_CUDA(cudaMemcpyAsync(p, out.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
}

int prob_check_desc(const double* p, int64_t n) {
  Stream st;
  Dev bad(sizeof(int));
  TNB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st.s));
  check_desc_kernel<<<grid_of(n), 256, 0, st.s>>>(p, n, (int*)bad.p);
  check_launch("check_desc");
  int h = 0;
  TNB_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
  return h;
}

void prob_prefix_at(const double* p, int64_t n, const int64_t* ks, int nk, double* sums) {
  if (n > (int64_t)INT32_MAX) throw Error(TNB_ERR_ARG, "scan size above 2^31");
  for (int i = 0; i < nk; ++i)
    if (ks[i] < 1 || ks[i] > n) throw Error(TNB_ERR_ARG, "prefix index out of range");
  Stream st;
  Dev cs(n * sizeof(double)), dk(nk * sizeof(int64_t)), dout(nk * sizeof(double));
  size_t tmp = 0;
  TNB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, p, (double*)cs.p, (int)n, st.s));
  Dev work(tmp);
  TNB_CUDA(cub::DeviceScan::InclusiveSum(work.p, tmp, p, (double*)cs.p, (int)n, st.s));
  TNB_CUDA(cudaMemcpyAsync(dk.p, ks, nk * sizeof(int64_t), cudaMemcpyHostToDevice, st.s));
  gather_kernel<<<(nk + 255) / 256, 256, 0, st.s>>>((const double*)cs.p, (const int64_t*)dk.p, nk,
                                                   (double*)dout.p);
  check_launch("prefix_at");
  TNB_CUDA(cudaMemcpyAsync(sums, dout.p, nk * sizeof(double), cudaMemcpyDeviceToHost, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
}

double prob_ks(const double* p_sorted_asc, int64_t n, double scale) {
  Stream st;
  Dev out(sizeof(unsigned long long));
  TNB_CUDA(cudaMemsetAsync(out.p, 0, sizeof(unsigned long long), st.s));
  ks_kernel<<<grid_of(n), 256, 0, st.s>>>(p_sorted_asc, n, scale, (unsigned long long*)out.p);
  check_launch("ks");
  unsigned long long h = 0;
  TNB_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st.s));
  TNB_CUDA(cudaStreamSynchronize(st.s));
  double d;
  memcpy(&d, &h, sizeof(d));
  return d;
}

}  // namespace tnb
