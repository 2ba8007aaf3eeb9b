/*
 * tnb.h -- C-ABI of the B200-native big-batch tensor-network contraction
 * executor (libtnb.so).  Plain pointers and sizes only; no torch types.
 *
 * The reference (`tncut` 0.1.0, /root/reference/pkg/src/tncut) has no FFI:
 * its hot path is the Python engine API.  Each entry point below replaces
 * one piece of that engine (file:line cite the reference):
 *
 *   tnb_program_create      -- the static part of `_contract_steps`
 *                              (engine.py:117-144) + `_split` (:171-185):
 *                              leaves, pairwise steps, sliced ids, root order
 *   tnb_program_set_leaf    -- `TensorNetwork.repin` (network.py:65-77) as seen
 *                              by the engine (`compute_head_vector` :259-260):
 *                              new leaf values, same topology
 *   tnb_program_run_range   -- `compute_head_vector`'s slice loop + sum
 *                              (engine.py:275-298): `_prepared_leaves`
 *                              (:102-114), `_contract_steps`, root transpose
 *                              (:287-290), `_fixed_tree_sum` (:207-222) /
 *                              free running sum (:295-298)
 *   tnb_program_run_range with n_sliced=0 -- `contract_tree` (engine.py:147-165)
 *                              and the tail contraction of
 *                              `compute_tail_amplitudes` (engine.py:358-377,
 *                              head-absorbed form)
 *   tnb_cgemm               -- one complex GEMM step (`np.tensordot` ->
 *                              `cgemm`, engine.py:129) on the tensor-core path
 *   tnb_add_tree            -- `reduce_partials`' aligned combine
 *                              (engine.py:428-442) on device buffers
 *
 * Error behaviour mirrors the reference's exceptions (errors.py):
 * every call returns a tnb_status; tnb_last_error() returns a thread-local
 * message.  The Python wrapper maps TNB_ERR_SHAPE -> ShapeMismatch
 * (errors.py:83-84), TNB_ERR_RANGE -> RangeOutOfBounds (:87-88),
 * TNB_ERR_ARG -> ValueError, everything else -> RuntimeError.
 */
#ifndef TNB_H
#define TNB_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TNB_ABI_VERSION 2

typedef enum {
  TNB_OK = 0,
  TNB_ERR_ARG = 1,      /* invalid argument (ValueError)                     */
  TNB_ERR_SHAPE = 2,    /* inconsistent network/steps (ShapeMismatch)         */
  TNB_ERR_RANGE = 3,    /* slice range outside [0, 2^n_e) (RangeOutOfBounds)  */
  TNB_ERR_CUDA = 4,     /* CUDA runtime/driver failure                        */
  TNB_ERR_NOMEM = 5,    /* device allocation failed                           */
  TNB_ERR_NODEV = 6     /* no sm_100 device                                   */
} tnb_status;

typedef enum { TNB_DOUBLE = 0, TNB_SINGLE = 1 } tnb_precision; /* engine.py:41 */
typedef enum { TNB_FIXED = 0, TNB_FREE = 1 } tnb_mode;          /* engine.py:293-300 */

/* program flags */
#define TNB_FLAG_NO_TENSOR_CORES 0x1u  /* force the SIMT contraction kernel      */
#define TNB_FLAG_NO_HOIST        0x2u  /* recompute slice-invariant subtrees     */
#define TNB_FLAG_REUSE_SLICES    0x4u  /* reuse results whose mask bits did not
                                          change between consecutive slices
                                          (bit-identical; skips recomputation)  */
#define TNB_FLAG_NO_FUSE         0x8u  /* stage every tensor-core operand with the
                                          permute/split kernel instead of writing
                                          it from the producer GEMM's epilogue   */

typedef struct tnb_program tnb_program;

typedef struct {
  int32_t n_leaves;
  const int64_t* leaf_ids;      /* node ids, n_leaves                               */
  const int32_t* leaf_ranks;    /* rank of each leaf (all bond dims are 2)          */
  const int64_t* leaf_indices;  /* concatenated index ids, leaf axis order          */
  const double* leaf_data;      /* concatenated interleaved complex128 values,
                                   2^rank per leaf, C order (network.py:30-39)      */
  int32_t n_steps;
  const int64_t* steps;         /* 3*n_steps: lhs, rhs, out (ordering.py:31-35)     */
  int32_t n_sliced;
  const int64_t* sliced;        /* MSB-first: bit (n_sliced-1-pos) of the mask pins
                                   sliced[pos] (engine.py:276-279)                  */
  int32_t n_out;
  const int64_t* out_order;     /* index ids of the root, in output axis order      */
  int32_t precision;            /* tnb_precision                                    */
  int32_t device;               /* CUDA device ordinal                              */
  uint32_t flags;               /* TNB_FLAG_*                                       */
} tnb_program_desc;

typedef struct {
  int64_t out_elems;            /* 2^n_out                                          */
  double flops_per_slice;       /* 8 * sum_steps 2^(n_A+n_B+n_AB)  (engine.py:455)  */
  double tc_flops_per_slice;    /* part of the above on the tensor-core path        */
  int64_t arena_bytes;          /* slice-variant intermediates                      */
  int64_t persistent_bytes;     /* leaves + hoisted slice-invariant results         */
  int64_t scratch_bytes;        /* largest per-step GEMM operand staging (in arena) */
  int32_t n_steps_tc;           /* steps on the tcgen05 path                        */
  int32_t n_steps_simt;         /* steps on the SIMT path                           */
  int32_t n_steps_hoisted;      /* slice-invariant steps computed once              */
  int32_t kernels_per_slice;    /* launches per slice                               */
  int64_t reuse_bytes;          /* TNB_FLAG_REUSE_SLICES: dedicated cached buffers  */
  int32_t n_steps_fused;        /* tensor-core steps whose result is written by the
                                   GEMM epilogue as the consumer's staged operand    */
  int32_t n_steps_fused_fast;   /* ... of which on the coalesced exchange path      */
} tnb_program_info;

typedef struct {
  double total_ms;              /* device time of the last run_range                */
  double gemm_ms;               /* tcgen05 GEMM kernels                             */
  double convert_ms;            /* permute/split operand staging kernels            */
  double simt_ms;               /* SIMT contraction kernels                         */
  double other_ms;              /* leaf gather, accumulate, root permute            */
  int64_t launches;             /* kernels launched by the last run_range           */
  int64_t gemm_launches;
  double gemm_flops;            /* algorithmic complex FLOPs executed on tcgen05    */
  int64_t steps_reused;         /* steps skipped by TNB_FLAG_REUSE_SLICES           */
  int64_t scale_redos;          /* fused producers re-run by the fp16 scale guard:
                                   the a-priori bound 2K max|A| max|B| was more than
                                   TNB_SCALE_GUARD_BITS (default 18) binary orders
                                   above the result's max (always counted)           */
} tnb_timing;

int tnb_abi_version(void);
const char* tnb_last_error(void);
int tnb_device_count(int32_t* n);

int tnb_program_create(const tnb_program_desc* desc, tnb_program** out);
int tnb_program_destroy(tnb_program* p);
int tnb_program_get_info(const tnb_program* p, tnb_program_info* info);

/* Replace one leaf's values (interleaved complex128 host data, 2^rank). */
int tnb_program_set_leaf(tnb_program* p, int32_t leaf_pos, const double* data);
/* Replace n leaves at once: data = their interleaved complex128 values
   concatenated in the order of `leaf_pos` (one staged upload, one sync). */
int tnb_program_set_leaves(tnb_program* p, int32_t n, const int32_t* leaf_pos,
                           const double* data);
/* Replace one leaf of a single-precision program from HOST complex64
   (interleaved float) data, no conversion. */
int tnb_program_set_leaf_c64(tnb_program* p, int32_t leaf_pos, const float* data);
/* Replace one leaf's values from DEVICE memory already in the program's
   precision (complex64 for single, complex128 for double). */
int tnb_program_set_leaf_device(tnb_program* p, int32_t leaf_pos, const void* dev_data);

/* Sum the contraction over slice masks [a, b) in `mode`, root permuted to
   out_order.  `out` receives 2^n_out complex values in the program's
   precision: host memory if out_on_device == 0, else device memory on the
   program's device.  Synchronous. */
int tnb_program_run_range(tnb_program* p, uint64_t a, uint64_t b, int32_t mode,
                          void* out, int32_t out_on_device);
/* CUDA-event timing of the next run_range calls: 0 off, 1 every kernel class
   (gemm/convert/simt/other), 2 GEMM launches + the range total only (no
   event records around the small kernels). */
int tnb_program_set_timing(tnb_program* p, int32_t enabled);
int tnb_program_get_timing(const tnb_program* p, tnb_timing* t);

/* C[M,N] = A[M,K] @ B[K,N], complex64, row-major, host or device pointers
   (`on_device`), on the tcgen05 3xFP16-split path when use_tc != 0 else
   the SIMT path.  Test/diagnostic entry for the per-step GEMM. */
int tnb_cgemm(int32_t device, int64_t M, int64_t N, int64_t K,
              const void* A, const void* B, void* C, int32_t on_device, int32_t use_tc);

/* out = sum of `n` device vectors (complex, `precision`) of `elems`
   entries along the aligned binary tree of reduce_partials
   (engine.py:428-442): ((v0+v1)+(v2+v3))+... for n a power of two,
   left-to-right otherwise.  Device pointers. */
int tnb_add_tree(int32_t device, int32_t precision, int64_t elems, int32_t n,
                 const void* const* vecs, void* out);

/* ---- On-device output-distribution analytics (tncut analytics.py) on a
   probability vector in device memory (`probs`, fp64).  Host results.
   Sums are deterministic (fixed reduction tree); counts/min/max exact. */

/* probs[i] = |amps[i]|^2 in fp64; amps complex64 (TNB_SINGLE) or complex128,
   the engine's AmplitudeTable.probabilities (engine.py:79-81). */
int tnb_probabilities(int32_t device, int32_t precision, const void* amps, int64_t n, double* probs);
/* out4 = {sum, min, max, min over p > 0 (+inf if none)}: the reductions of
   xeb (analytics.py:46-58), marginal_and_conditional (:159-177) and the
   log-scale histogram range (:104-107). */
int tnb_prob_reduce(int32_t device, const double* probs, int64_t n, double* out4_host);
/* counts of x = scale * p per bin [edges[i], edges[i+1]) (last bin closed),
   np.histogram semantics of histogram() (analytics.py:90-121). */
int tnb_prob_histogram(int32_t device, const double* probs, int64_t n, double scale,
                       const double* edges_host, int32_t bins, int64_t* counts_host);
/* in-place radix sort (ascending, or descending if `descending`). */
int tnb_prob_sort(int32_t device, double* probs, int64_t n, int32_t descending);
/* sortedness check of postselect_curve (analytics.py:136-137). */
int tnb_prob_is_sorted_desc(int32_t device, const double* probs, int64_t n, int32_t* sorted_host);
/* sums_host[j] = probs[0] + ... + probs[ks[j]-1] (the cumsum of
   postselect_curve, analytics.py:138-142). */
int tnb_prob_prefix_sums(int32_t device, const double* probs, int64_t n, const int64_t* ks_host,
                         int32_t nk, double* sums_host);
/* KS distance of scale * p (sorted ascending) against Exp(1)
   (ks_to_porter_thomas, analytics.py:70-79). */
int tnb_prob_ks(int32_t device, const double* probs_sorted_asc, int64_t n, double scale,
                double* out_host);

/* ---- The multi-GPU path's one collective: a sum over ranks of
   the amplitude (or head-vector) partials of disjoint slice ranges, over
   NCCL (libnccl.so.2 is dlopen'd on first use; no link-time dependency).
   One communicator per process/device; `stream` NULL = the legacy stream.
   Reference interface replaced: the reference has no collective -- partial
   head vectors travel as TNCUTHV1 files and are summed by reduce_partials
   (engine.py:398-452, cli.py:417-441). */
int tnb_nccl_unique_id(uint8_t id_out[128]);
int tnb_nccl_comm_create(int32_t nranks, const uint8_t id[128], int32_t rank, int32_t device,
                         void** comm_out);
int tnb_nccl_comm_destroy(void* comm);
/* in-place sum of n complex values (complex64 if TNB_SINGLE, complex128
   otherwise) in device memory; returns after the collective completed. */
int tnb_allreduce_sum(void* comm, int32_t precision, void* dev_buf, int64_t n_complex,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TNB_H */
