// extern "C" boundary of libtnb.so (declared in include/tnb.h).  Converts
// tnb::Error into status codes + a thread-local message, as the reference's
// engine raises errors.py exceptions (see tnb.h for the mapping).
#include "tnb_internal.h"

#include <cstring>
#include <functional>
#include <memory>

namespace tnb {

struct Program;
Program* program_create(const tnb_program_desc* d);
void program_destroy(Program* P);
void program_info(const Program* P, tnb_program_info* info);
void program_set_leaf(Program* P, int leaf_pos, const double* data);
void program_set_leaf_device(Program* P, int leaf_pos, const void* dev);
void program_set_leaves(Program* P, int n, const int32_t* pos, const double* data);
void program_set_leaf_c64(Program* P, int leaf_pos, const float* data);
void program_run_range(Program* P, uint64_t a, uint64_t b, int mode, void* out, int out_dev);
void program_set_timing(Program* P, int on);
void program_get_timing(const Program* P, tnb_timing* t);
// analytics.cu
void prob_from_amps(int precision, const void* amps, int64_t n, double* p);
void prob_reduce(const double* p, int64_t n, double* out4);
void prob_histogram(const double* p, int64_t n, double scale, const double* edges, int bins, int64_t* counts);
void prob_sort(double* p, int64_t n, int descending);
int prob_check_desc(const double* p, int64_t n);
void prob_prefix_at(const double* p, int64_t n, const int64_t* ks, int nk, double* sums);
double prob_ks(const double* p_sorted_asc, int64_t n, double scale);

namespace {
thread_local std::string g_err;
}
void set_last_error(const std::string& m) { g_err = m; }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return TNB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return TNB_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TNB_ERR_ARG;
  }
}

// owning device buffer
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t n) { TNB_CUDA(cudaMalloc(&p, n ? n : 16)); }
  ~DevBuf() { if (p) cudaFree(p); }
};

}  // namespace tnb

using namespace tnb;

extern "C" {

int tnb_abi_version(void) { return TNB_ABI_VERSION; }

const char* tnb_last_error(void) { return g_err.c_str(); }

int tnb_device_count(int32_t* n) {
  return guarded([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) c = 0;
    *n = c;
  });
}

int tnb_program_create(const tnb_program_desc* desc, tnb_program** out) {
  return guarded([&] {
    if (!out) throw Error(TNB_ERR_ARG, "null output handle");
    *out = reinterpret_cast<tnb_program*>(program_create(desc));
  });
}

int tnb_program_destroy(tnb_program* p) {
  return guarded([&] { program_destroy(reinterpret_cast<Program*>(p)); });
}

int tnb_program_get_info(const tnb_program* p, tnb_program_info* info) {
  return guarded([&] {
    if (!p || !info) throw Error(TNB_ERR_ARG, "null argument");
    program_info(reinterpret_cast<const Program*>(p), info);
  });
}

int tnb_program_set_leaf(tnb_program* p, int32_t leaf_pos, const double* data) {
  return guarded([&] {
    if (!p || !data) throw Error(TNB_ERR_ARG, "null argument");
    program_set_leaf(reinterpret_cast<Program*>(p), leaf_pos, data);
  });
}

int tnb_program_set_leaves(tnb_program* p, int32_t n, const int32_t* leaf_pos, const double* data) {
  return guarded([&] {
    if (!p || (n > 0 && (!leaf_pos || !data))) throw Error(TNB_ERR_ARG, "null argument");
    program_set_leaves(reinterpret_cast<Program*>(p), n, leaf_pos, data);
  });
}

int tnb_program_set_leaf_c64(tnb_program* p, int32_t leaf_pos, const float* data) {
  return guarded([&] {
    if (!p || !data) throw Error(TNB_ERR_ARG, "null argument");
    program_set_leaf_c64(reinterpret_cast<Program*>(p), leaf_pos, data);
  });
}

int tnb_program_set_leaf_device(tnb_program* p, int32_t leaf_pos, const void* dev_data) {
  return guarded([&] {
    if (!p || !dev_data) throw Error(TNB_ERR_ARG, "null argument");
    program_set_leaf_device(reinterpret_cast<Program*>(p), leaf_pos, dev_data);
  });
}

int tnb_program_run_range(tnb_program* p, uint64_t a, uint64_t b, int32_t mode, void* out,
                          int32_t out_on_device) {
  return guarded([&] {
    if (!p) throw Error(TNB_ERR_ARG, "null program");
    program_run_range(reinterpret_cast<Program*>(p), a, b, mode, out, out_on_device);
  });
}

int tnb_program_set_timing(tnb_program* p, int32_t enabled) {
  return guarded([&] {
    if (!p) throw Error(TNB_ERR_ARG, "null program");
    program_set_timing(reinterpret_cast<Program*>(p), enabled);
  });
}

int tnb_program_get_timing(const tnb_program* p, tnb_timing* t) {
  return guarded([&] {
    if (!p || !t) throw Error(TNB_ERR_ARG, "null argument");
    program_get_timing(reinterpret_cast<const Program*>(p), t);
  });
}

int tnb_cgemm(int32_t device, int64_t M, int64_t N, int64_t K, const void* A, const void* B,
              void* C, int32_t on_device, int32_t use_tc) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0) throw Error(TNB_ERR_ARG, "GEMM dims must be positive");
    if (M * K > (1ll << 32) || K * N > (1ll << 32) || M * N > (1ll << 32))
      throw Error(TNB_ERR_ARG, "GEMM operand above 2^32 elements");
    TNB_CUDA(cudaSetDevice(device));
    int sms = 148;
    TNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t st;
    TNB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SD { cudaStream_t s; ~SD() { cudaStreamDestroy(s); } } sd{st};
    const size_t ea = (size_t)(M * K) * 8, eb = (size_t)(K * N) * 8, ec = (size_t)(M * N) * 8;
    std::unique_ptr<DevBuf> da, db, dc;
    const void* pa = A;
    const void* pb = B;
    void* pc = C;
    if (!on_device) {
      da.reset(new DevBuf(ea)); db.reset(new DevBuf(eb)); dc.reset(new DevBuf(ec));
      TNB_CUDA(cudaMemcpyAsync(da->p, A, ea, cudaMemcpyHostToDevice, st));
      TNB_CUDA(cudaMemcpyAsync(db->p, B, eb, cudaMemcpyHostToDevice, st));
      pa = da->p; pb = db->p; pc = dc->p;
    }
    // A is [M][K] row-major: canonical (m,k) identity.  B is [K][N]: canonical
    // (n,k) index n*K+k lives at k*N+n.
    auto bits_of = [](int64_t v) { int b = 0; while ((1ll << b) < v) ++b; return b; };
    const int bm = bits_of(M), bn = bits_of(N), bk = bits_of(K);
    if ((1ll << bm) != M || (1ll << bn) != N || (1ll << bk) != K)
      throw Error(TNB_ERR_ARG, "GEMM dims must be powers of two");
    std::vector<int> la, lb;
    for (int p = 0; p < bk + bm; ++p) la.push_back(p);
    for (int p = 0; p < bk; ++p) lb.push_back(bn + p);   // k bits sit above n bits in B
    for (int p = 0; p < bn; ++p) lb.push_back(p);
    const bool tc = use_tc && tc_available(device);
    if (use_tc && !tc) throw Error(TNB_ERR_NODEV, "tensor-core path needs an sm_100 device");
    if (!tc) {
      ByteLut hl[2];
      build_lut(la, &hl[0]);
      build_lut(lb, &hl[1]);
      DevBuf dl(sizeof(hl));
      TNB_CUDA(cudaMemcpyAsync(dl.p, hl, sizeof(hl), cudaMemcpyHostToDevice, st));
      const ByteLut* lut = (const ByteLut*)dl.p;
      launch_contract_simt<float2>((const float2*)pa, (const float2*)pb, (float2*)pc, M, N, K, lut,
                                   lut + 1, nullptr, nullptr, nullptr, st);
      TNB_CUDA(cudaStreamSynchronize(st));
    } else {
      const int64_t Kp = 2 * K, Np = 2 * N;
      const int64_t ws = tc_workspace_elems(M, Np, Kp, sms);
      DevBuf scratch((size_t)(2 * M * Kp + 2 * Np * Kp) * 2 + 1024 + (size_t)ws * 4);
      DevBuf maxbits(64);
      TNB_CUDA(cudaMemsetAsync(maxbits.p, 0, 64, st));
      unsigned* mx = (unsigned*)maxbits.p;
      __half* ahi = (__half*)scratch.p;
      __half* alo = ahi + M * Kp;
      __half* bhi = alo + M * Kp;
      __half* blo = bhi + Np * Kp;
      float* wsp = (float*)((char*)scratch.p + (((size_t)(2 * M * Kp + 2 * Np * Kp) * 2 + 1023) / 1024) * 1024);
      StageHost sh[2];
      build_stage_tables(la, K, &sh[0]);
      build_stage_tables(lb, K, &sh[1]);
      std::vector<std::unique_ptr<DevBuf>> keep;
      StageTables tb[2];
      for (int i = 0; i < 2; ++i) {
        const size_t n = sh[i].rd_t.size();
        keep.emplace_back(new DevBuf(3 * n * 4 + 2 * sizeof(ByteLut)));
        char* b = (char*)keep.back()->p;
        TNB_CUDA(cudaMemcpyAsync(b, sh[i].rd_t.data(), n * 4, cudaMemcpyHostToDevice, st));
        TNB_CUDA(cudaMemcpyAsync(b + n * 4, sh[i].rd_src.data(), n * 4, cudaMemcpyHostToDevice, st));
        TNB_CUDA(cudaMemcpyAsync(b + 2 * n * 4, sh[i].t_dst.data(), n * 4, cudaMemcpyHostToDevice, st));
        TNB_CUDA(cudaMemcpyAsync(b + 3 * n * 4, &sh[i].tile_src, sizeof(ByteLut), cudaMemcpyHostToDevice, st));
        TNB_CUDA(cudaMemcpyAsync(b + 3 * n * 4 + sizeof(ByteLut), &sh[i].tile_dst, sizeof(ByteLut),
                                 cudaMemcpyHostToDevice, st));
        tb[i].rd_t = (const uint32_t*)b;
        tb[i].rd_src = (const uint32_t*)(b + n * 4);
        tb[i].t_dst = (const uint32_t*)(b + 2 * n * 4);
        tb[i].tile_src = (const ByteLut*)(b + 3 * n * 4);
        tb[i].tile_dst = (const ByteLut*)(b + 3 * n * 4 + sizeof(ByteLut));
        tb[i].nU = sh[i].nU;
        tb[i].n_tiles = sh[i].n_tiles;
      }
      launch_absmax((const float2*)pa, M * K, mx, st);
      launch_absmax((const float2*)pb, N * K, mx + 1, st);
      launch_stage((const float2*)pa, tb[0], K, false, mx, ahi, alo, st);
      launch_stage((const float2*)pb, tb[1], K, true, mx + 1, bhi, blo, st);
      TcGemmPlan plan;
      ScaleSrc sa, sb;
      sa.a = mx;
      sb.a = mx + 1;
      tc_plan_gemm(&plan, ahi, alo, bhi, blo, M, Np, Kp, (float*)pc, wsp, ws, sa, sb, mx + 2, sms);
      DevBuf progress((size_t)sms * 4);
      plan.progress = (unsigned int*)progress.p;
      tc_launch_gemm(&plan, st);
      if (plan.splits > 1)
        launch_splitk_reduce(plan.C, plan.splits, M * Np, (float*)pc, sa, sb, mx + 2, st);
      TNB_CUDA(cudaStreamSynchronize(st));
    }
    if (!on_device) TNB_CUDA(cudaMemcpyAsync(C, pc, ec, cudaMemcpyDeviceToHost, st));
    TNB_CUDA(cudaStreamSynchronize(st));
  });
}

int tnb_add_tree(int32_t device, int32_t precision, int64_t elems, int32_t n,
                 const void* const* vecs, void* out) {
  return guarded([&] {
    if (n <= 0 || !vecs || !out) throw Error(TNB_ERR_ARG, "bad add_tree arguments");
    TNB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    TNB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SD { cudaStream_t s; ~SD() { cudaStreamDestroy(s); } } sd{st};
    const bool pow2 = (n & (n - 1)) == 0;
    const size_t es = precision == TNB_SINGLE ? 8 : 16;
    // scratch per recursion level
    std::vector<std::unique_ptr<DevBuf>> tmp;
    std::function<const void*(int, int)> combine = [&](int lo, int hi) -> const void* {
      if (hi - lo == 1) return vecs[lo];
      const int mid = (lo + hi) / 2;
      const void* l = combine(lo, mid);
      const void* r = combine(mid, hi);
      tmp.emplace_back(new DevBuf((size_t)elems * es));
      void* o = tmp.back()->p;
      if (precision == TNB_SINGLE) launch_add<float2>((const float2*)l, (const float2*)r, (float2*)o, elems, st);
      else launch_add<double2>((const double2*)l, (const double2*)r, (double2*)o, elems, st);
      return o;
    };
    const void* res;
    if (pow2) {
      res = combine(0, n);
    } else {
      // unaligned: deterministic left fold (reduce_partials fallback, engine.py:443-447)
      res = vecs[0];
      for (int i = 1; i < n; ++i) {
        tmp.emplace_back(new DevBuf((size_t)elems * es));
        void* o = tmp.back()->p;
        if (precision == TNB_SINGLE) launch_add<float2>((const float2*)res, (const float2*)vecs[i], (float2*)o, elems, st);
        else launch_add<double2>((const double2*)res, (const double2*)vecs[i], (double2*)o, elems, st);
        res = o;
      }
    }
    TNB_CUDA(cudaMemcpyAsync(out, res, (size_t)elems * es, cudaMemcpyDeviceToDevice, st));
    TNB_CUDA(cudaStreamSynchronize(st));
  });
}


// ---- on-device analytics (analytics.py); all pointers are device pointers
// on `device` unless named *_host
int tnb_probabilities(int32_t device, int32_t precision, const void* amps, int64_t n, double* probs) {
  return guarded([&] {
    if (!amps || !probs || n < 0) throw Error(TNB_ERR_ARG, "bad probabilities arguments");
    TNB_CUDA(cudaSetDevice(device));
    if (n) prob_from_amps(precision, amps, n, probs);
  });
}

int tnb_prob_reduce(int32_t device, const double* probs, int64_t n, double* out4_host) {
  return guarded([&] {
    if (!probs || !out4_host || n <= 0) throw Error(TNB_ERR_ARG, "bad reduce arguments");
    TNB_CUDA(cudaSetDevice(device));
    prob_reduce(probs, n, out4_host);
  });
}

int tnb_prob_histogram(int32_t device, const double* probs, int64_t n, double scale,
                       const double* edges_host, int32_t bins, int64_t* counts_host) {
  return guarded([&] {
    if (!probs || !edges_host || !counts_host || n <= 0) throw Error(TNB_ERR_ARG, "bad histogram arguments");
    TNB_CUDA(cudaSetDevice(device));
    prob_histogram(probs, n, scale, edges_host, bins, counts_host);
  });
}

int tnb_prob_sort(int32_t device, double* probs, int64_t n, int32_t descending) {
  return guarded([&] {
    if (!probs || n < 0) throw Error(TNB_ERR_ARG, "bad sort arguments");
    TNB_CUDA(cudaSetDevice(device));
    if (n > 1) prob_sort(probs, n, descending);
  });
}

int tnb_prob_is_sorted_desc(int32_t device, const double* probs, int64_t n, int32_t* sorted_host) {
  return guarded([&] {
    if (!probs || !sorted_host || n < 0) throw Error(TNB_ERR_ARG, "bad sortedness arguments");
    TNB_CUDA(cudaSetDevice(device));
    *sorted_host = n > 1 ? !prob_check_desc(probs, n) : 1;
  });
}

int tnb_prob_prefix_sums(int32_t device, const double* probs, int64_t n, const int64_t* ks_host,
                         int32_t nk, double* sums_host) {
  return guarded([&] {
    if (!probs || !ks_host || !sums_host || n <= 0 || nk <= 0) throw Error(TNB_ERR_ARG, "bad prefix arguments");
    TNB_CUDA(cudaSetDevice(device));
    prob_prefix_at(probs, n, ks_host, nk, sums_host);
  });
}

int tnb_prob_ks(int32_t device, const double* probs_sorted_asc, int64_t n, double scale, double* out_host) {
  return guarded([&] {
    if (!probs_sorted_asc || !out_host || n <= 0) throw Error(TNB_ERR_ARG, "bad ks arguments");
    TNB_CUDA(cudaSetDevice(device));
    *out_host = prob_ks(probs_sorted_asc, n, scale);
  });
}

int tnb_nccl_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    if (!id_out) throw Error(TNB_ERR_ARG, "null id buffer");
    nccl_unique_id(id_out);
  });
}

int tnb_nccl_comm_create(int32_t nranks, const uint8_t id[128], int32_t rank, int32_t device,
                         void** comm_out) {
  return guarded([&] {
    if (!id || !comm_out) throw Error(TNB_ERR_ARG, "null NCCL argument");
    *comm_out = nccl_comm_create(nranks, id, rank, device);
  });
}

int tnb_nccl_comm_destroy(void* comm) {
  return guarded([&] { nccl_comm_destroy(comm); });
}

int tnb_allreduce_sum(void* comm, int32_t precision, void* dev_buf, int64_t n_complex, void* stream) {
  return guarded([&] {
    if (precision != TNB_SINGLE && precision != TNB_DOUBLE) throw Error(TNB_ERR_ARG, "bad precision");
    nccl_allreduce_sum(comm, precision, dev_buf, n_complex, stream);
  });
}

}  // extern "C"
