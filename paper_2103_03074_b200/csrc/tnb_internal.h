// Internal declarations shared by the libtnb translation units.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <string>
#include <vector>
#include <stdexcept>

#include "../../include/tnb.h"

namespace tnb {

// ---------------------------------------------------------------------------
// Errors: every internal failure throws tnb::Error(code, msg); the C-ABI
// layer converts it into a status + thread-local message.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& m);

#define TNB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      throw ::tnb::Error(_e == cudaErrorMemoryAllocation ? TNB_ERR_NOMEM : TNB_ERR_CUDA, \
                         std::string(#call) + ": " + cudaGetErrorString(_e));       \
    }                                                                               \
  } while (0)

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(TNB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Byte lookup tables that map a canonical (row-major GEMM) element index to
// the element offset inside a tensor stored with an arbitrary axis order.
// All bond dimensions are 2, so an index is a bit vector and the map is a
// bit permutation: src = T0[j & 255] | T1[(j>>8)&255] | T2[(j>>16)&255] | T3[j>>24].
struct ByteLut {
  uint32_t t[4][256];
};

// Build the LUT for a permutation given as src_bit[p] = source bit position
// of canonical bit p (p = 0 is the least significant canonical bit).
void build_lut(const std::vector<int>& src_bit, ByteLut* out);

// ---------------------------------------------------------------------------
// fp16 split scale of a staged operand: s = 2^(15-e) where the bound
// v = f * max(a) [* max(b)] = frac * 2^e (frac in [0.5, 1)), so v*s lands in
// [2^14, 2^15).  Staged operands use their own exact max (b = null, f = 1);
// operands written by the producer's epilogue (fused staging) use the a-priori
// bound |x| <= 2 K max|A| max|B| of the producing step (its operands' maxes),
// known before the producer runs.
struct ScaleSrc {
  const unsigned int* a = nullptr;
  const unsigned int* b = nullptr;
  float f = 1.f;  // power of two
  // runtime guard of a fused operand (consumer side): when *guard != 0 the
  // producer was re-run with its result's exact max (`own`) as the scale
  // source because the a-priori bound was looser than the guard threshold
  const unsigned int* guard = nullptr;
  const unsigned int* own = nullptr;
};

#ifdef __CUDACC__
// exponent e of the scale source's bound v = frac * 2^e (frac in [0.5, 1));
// false when the bound is zero (all-zero operand)
__device__ __forceinline__ bool scale_bound_exp(const unsigned int* pa, const unsigned int* pb,
                                                float f, int& e) {
  const float ma = __uint_as_float(*pa);
  if (!(ma > 0.f)) return false;
  float fr = frexpf(ma, &e);  // ma = fr * 2^e
  if (pb != nullptr) {
    const float mb = __uint_as_float(*pb);
    if (!(mb > 0.f)) return false;
    int eb, ef, ep;
    const float fb = frexpf(mb, &eb);
    frexpf(f, &ef);              // f = 2^(ef-1)
    fr = frexpf(fr * fb, &ep);   // product of the fractions in [0.25, 1)
    e = e + eb + (ef - 1) + ep;
  } else if (f != 1.f) {
    int ef;
    frexpf(f, &ef);
    e += ef - 1;
  }
  return true;
}

__device__ __forceinline__ float scale_from_src(const ScaleSrc& s) {
  int e;
  const bool own = s.guard != nullptr && *s.guard != 0u;
  if (!(own ? scale_bound_exp(s.own, nullptr, 1.f, e) : scale_bound_exp(s.a, s.b, s.f, e)))
    return 1.f;
  int p = 15 - e;
  p = p > 126 ? 126 : (p < -126 ? -126 : p);
  return ldexpf(1.f, p);
}
#endif


// ---------------------------------------------------------------------------
// Kernel launchers (kernels.cu).  All take a stream; pointers are device.
struct SlicedLeafDesc {      // one sliced leaf to prepare per mask
  uint64_t src_off;          // element offset of the full leaf in the leaf pool
  uint64_t dst_off;          // element offset of the prepared leaf (slice pool)
  uint32_t out_elems;        // 2^(rank - #sliced axes)
  uint32_t n_sl;             // number of sliced axes (<= 8)
  uint32_t keep_lut_off;     // offset into a shared uint32 table: out index -> src offset
  uint32_t pad;
  uint32_t sl_stride[8];     // element stride of each sliced axis in the full leaf
  uint32_t sl_bit[8];        // mask bit position (n_e-1-pos)
};

template <typename T>
void launch_prepare_leaves(const T* leaf_pool, T* slice_pool, const SlicedLeafDesc* descs,
                           int n_descs, const uint32_t* keep_tables, uint64_t mask,
                           cudaStream_t s);

struct FuseOut;
// C = A B over the gathered layouts; `fuse` (single precision, small-K kernel
// only, may be null): write C as a tensor-core consumer's staged operand
template <typename T>
// lutE (small-K kernel only, may be null): thread-quad -> output-quad enumeration
void launch_contract_simt(const T* A, const T* B, T* C, int64_t M, int64_t N, int64_t K,
                          const ByteLut* lutA, const ByteLut* lutB, const ByteLut* lutE,
                          unsigned int* max_out, const FuseOut* fuse, cudaStream_t s);
// one step of a batched SIMT launch (contract_simt_batch_kernel)
struct SimtStepDesc {
  const void* A;
  const void* B;
  void* C;
  int64_t M, N, K;
  const ByteLut* lut_a;
  const ByteLut* lut_b;
  unsigned int* max_out;
  int64_t block0;             // first block of this step in the batch grid
};
int64_t simt_tiles(int64_t M, int64_t N);
template <typename T>
void launch_contract_simt_batch(const SimtStepDesc* descs, int n, int64_t blocks, cudaStream_t s);
// whether launch_contract_simt takes the streaming small-K kernel
inline bool simt_uses_smallk(int64_t M, int64_t N, int64_t K) {
  return K <= 8 && N >= 4 && M * N >= (1 << 16);
}
// ... or the 64x64-tile kernel (4x4 outputs per thread; the big steps of the
// fp64 path, which has no tensor-core mode); never batched
inline bool simt_uses_wide(int64_t M, int64_t N, int64_t K) {
  return !simt_uses_smallk(M, N, K) && M >= 64 && N >= 64 && K >= 16;
}

template <typename T>
void launch_permute(const T* in, T* out, int64_t elems, const ByteLut* lut, cudaStream_t s);

template <typename T>
void launch_counter_merge(const T* x, const T* slots, int64_t stride, int n_merge, T* dst,
                          int64_t elems, cudaStream_t s);

template <typename T>
void launch_add(const T* a, const T* b, T* out, int64_t elems, cudaStream_t s);

template <typename T>
void launch_copy(const T* a, T* out, int64_t elems, cudaStream_t s);

// Tensor-core operand staging (single precision only).  Every single-
// precision tensor carries a device max|re|,|im| slot (fp32 bits) written by
// its producer; the staging kernels derive the power-of-two fp16 scale from it.
void launch_absmax(const float2* A, int64_t n, unsigned int* maxbits, cudaStream_t s);

// Tiled permute tables for one operand (see stage_kernel in kernels.cu).
struct StageHost {
  int nU = 0;
  int64_t n_tiles = 0;
  std::vector<uint32_t> rd_t, rd_src, t_dst;
  ByteLut tile_src, tile_dst;
};
struct StageTables {  // device view
  const uint32_t* rd_t;
  const uint32_t* rd_src;
  const uint32_t* t_dst;
  const ByteLut* tile_src;
  const ByteLut* tile_dst;
  int nU;
  int64_t n_tiles;
};
// Staged operands are K-blocked: [K / 2^kKBlockLog][rows][2^kKBlockLog]
// complex elements (one GEMM K block = 32 fp16 = 64 B per row), so every
// TMA box of the GEMM is one contiguous 8 KB read.  When K <= 2^kKBlockLog
// this is plain row-major [rows][K].
constexpr int kKBlockLog = 4;
// canon_to_src[p] = source bit of canonical (row*K + k) bit p
void build_stage_tables(const std::vector<int>& canon_to_src, int64_t K, StageHost* out);
void launch_stage(const float2* src, const StageTables& tb, int64_t K, bool expand,
                  const unsigned int* maxbits, __half* hi, __half* lo, cudaStream_t s);
void launch_splitk_reduce(const float* ws, int splits, int64_t elems, float* C,
                          const ScaleSrc& scale_rows, const ScaleSrc& scale_cols,
                          unsigned int* max_out, cudaStream_t s);

// Fused staging: the producer GEMM's epilogue writes its result straight into
// the consumer GEMM's operand layout (K-blocked fp16 hi/lo planes; role 1 =
// the consumer's rows operand, role 2 = its 2x2-expanded cols operand).  The
// destination half2 index of result element (m, n) is lut_m(m) | lut_n(n)
// (a bit permutation); dlow[j] = lut_n(j) for the 32 columns of one thread.
//
// Fast path (`fast`): one thread holds row m (lane = m bits 0-4) and 32
// complex columns (n bits 0-4 = vector element e (2 bits) | slot q (3 bits)).
// When n bits 0,1 are destination bits 0,1, up to three butterfly exchanges
// (slot bit j <-> lane bit log2(xlane[j])) move the source bits whose
// destination bits are lowest onto the lanes, so each warp store writes
// contiguous runs; the address is then tile base | lane part | slot_w[q].
struct FuseOut {
  int mode = 0;                  // 0: plain fp32 C; 1: rows operand; 2: cols operand
  int L = 0;                     // cols: rows 2n / 2n+1 are 2^L half2 apart
  int fast = 0;                  // GEMM epilogue: exchange + 16-B store path usable
  int vec = 0;                   // small-K SIMT producer: n bits 0,1 -> destination bits 0,1
  int xlane[3] = {0, 0, 0};      // lane xor mask exchanged with slot bit j (0: none)
  uint32_t lane_w[5] = {};       // destination weight of lane bit b (after exchanges)
  uint32_t slot_w[8] = {};       // destination offset of slot q (after exchanges)
  int nslot = 8;                 // fast path: 4-complex slots per thread (8, or 4 at 16 columns)
  __half2* hi = nullptr;
  __half2* lo = nullptr;
  const ByteLut* lut_m = nullptr;
  const ByteLut* lut_n = nullptr;
  uint32_t dlow[32] = {};
  ScaleSrc scale;                // scale of the written operand
  // fp16 scale guard re-run of a fused producer (redo != 0): every CTA first
  // decides whether the a-priori bound `guard_bound` exceeds the result's
  // exact max (scale.a, published by the first run) by more than guard_bits
  // binary orders; CTA 0 records the decision in *guard_word (read by the
  // consumer's ScaleSrc) and counts it; without it the launch exits at once
  int redo = 0;
  int guard_bits = 18;
  ScaleSrc guard_bound;
  unsigned int* guard_word = nullptr;
  unsigned int* guard_count = nullptr;
};

#ifdef __CUDACC__
// the re-run prologue (see FuseOut::redo); true = rewrite the operand
__device__ __forceinline__ bool fused_redo_fires(const FuseOut& fo) {
  const float mo = __uint_as_float(__ldcg(fo.scale.a));
  int eb = 0, eo = 0;
  bool fire = false;
  if (mo > 0.f && scale_bound_exp(fo.guard_bound.a, fo.guard_bound.b, fo.guard_bound.f, eb)) {
    frexpf(mo, &eo);
    fire = (eb - eo) > fo.guard_bits;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *fo.guard_word = fire ? 1u : 0u;
    if (fire) atomicAdd(fo.guard_count, 1u);
  }
  return fire;
}
#endif

// ---------------------------------------------------------------------------
// tcgen05 GEMM (gemm_tc.cu):  C[M][Np] (fp32) = alpha * sum over the three
// split products of Ahi/Alo[M][Kp] (fp16, K-major) x Bhi/Blo[Np][Kp].
struct TcGemmPlan {
  int64_t M = 0, Np = 0, Kp = 0;
  const __half* ahi = nullptr;   // staged operand planes (also in the TMA maps): the
  const __half* alo = nullptr;   // short-K skinny path reads them directly
  const __half* bhi = nullptr;
  const __half* blo = nullptr;
  int skinny = 0;                // Kp <= 32 and Np <= 64: FP32-pipe kernel instead of tcgen05
  int splits = 1;
  int chunk_kb = 8;              // promotion chunk (K blocks); see gemm_tc.cu
  int group_m = 16;              // raster band height (m-tiles)
  int cta_group = 1;             // 1: one CTA per 128x256 tile; 2: CTA pair per 256x256 tile
  int nb = 256;                  // tile width (accumulator columns): 64 / 128 / 256
  unsigned int* progress = nullptr;  // device [num units]: K-block progress for soft pacing
  int pace_slack = 0;            // K blocks a unit may lead the slowest one (0: off)
  int epi_spin = 0;              // epilogue polls the TMEM-ready barrier instead of sleeping
  int64_t k_per_split = 0;       // multiple of the K block
  int grid = 0;
  alignas(64) unsigned char tmap[4][128];  // CUtensorMap x4: Ahi, Alo, Bhi, Blo
  float* C = nullptr;            // output (splits == 1) or workspace [splits][M][Np]
  ScaleSrc scale_rows;           // fp16 split scale of the rows operand
  ScaleSrc scale_cols;           // ... and of the cols operand
  unsigned int* max_out = nullptr;         // device: max bits of the result (atomicMax)
  FuseOut fuse;                  // epilogue output format (splits == 1 only)
};

bool tc_available(int device);
void tc_plan_gemm(TcGemmPlan* p, const __half* Ahi, const __half* Alo, const __half* Bhi,
                  const __half* Blo, int64_t M, int64_t Np, int64_t Kp, float* C,
                  float* workspace, int64_t workspace_elems, const ScaleSrc& scale_rows,
                  const ScaleSrc& scale_cols, unsigned int* max_out, int num_sms);
void tc_launch_gemm(const TcGemmPlan* p, cudaStream_t s);
int64_t tc_workspace_elems(int64_t M, int64_t Np, int64_t Kp, int num_sms);
int tc_splits(int64_t M, int64_t Np, int64_t Kp, int num_sms);

// collective.cu: NCCL (dlopen'd) sum over ranks of complex partials
void nccl_unique_id(uint8_t* out128);
void* nccl_comm_create(int nranks, const uint8_t* id128, int rank, int device);
void nccl_comm_destroy(void* comm);
void nccl_allreduce_sum(void* comm, int precision, void* buf, int64_t n_complex, void* stream);

}  // namespace tnb
