/* tnb_plan.h -- C-ABI of the host-side head-tree / slice co-optimiser
 * (libtnbplan.so, paper_2103_03074_b200/csrc/treeopt.cpp).
 *
 * Replaces, for the head side of a first-cut tree, the reference's slice
 * selection `select_slices(tn, tree, target_space, reconfigure=True)`
 * (tncut/slicing.py:76-196) and its greedy subtree rebuild
 * `_reconfigure_once` (slicing.py:199-251, which reuses the greedy pair
 * order of ordering.py:256-285).  The reference has no FFI; the Python
 * mirror is paper_2103_03074_b200.treeopt.select_slices_b200, which returns
 * the reference's own (SlicePlan, ContractionTree) pair.
 *
 * Network encoding: head leaves 0..n-1 with their index ids (dense
 * 0..n_index-1) in CSR form (leaf_ptr[n+1], leaf_idx[]); every index has at
 * most two endpoints among the leaves (one = a cut leg that stays open).
 * Tree encoding (SSA): internal node n+i has children children[2i],
 * children[2i+1] (ids < n+i for the emitted tree), the root is 2n-2.
 */
#ifndef TNB_PLAN_H
#define TNB_PLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int target_log2;      /* max tensor rank after slicing (space target)    */
  int trials;           /* random-greedy trees                              */
  int keep_top;         /* cheapest trees carried into slicing              */
  int reconf_k;         /* subtree frontier size while slicing              */
  int polish_k;         /* subtree frontier size of the final polish        */
  int threads;          /* 0 = all hardware threads                         */
  int objective;        /* 0 = multiplications (engine.py:138-140 counter), */
                        /* 1 = B200 time model max(8*mults/F, bytes/BW)+t0  */
  uint64_t seed;
  double gemm_flops;    /* model F: complex-algorithmic FLOP/s of a step    */
  double hbm_bytes;     /* model BW: bytes/s of operand + result traffic    */
  double step_s;        /* model t0: fixed seconds per step                 */
  double time_budget_s; /* soft wall-clock budget                           */
  int slice_repeats;    /* slicing runs per tree (1st greedy, rest noisy)   */
  int keep_slices;      /* 1: init_sliced is kept as is; only the caller's  */
                        /*    tree is re-optimised (same slices, new order) */
} tnbp_options;

void tnbp_default_options(tnbp_options* opt);

/* Optimise the head tree and its sliced-index set for the total head work
 * 2^n_sliced * cost(one slice) with every tensor of rank <= target_log2.
 * init_children (nullable): the caller's tree, always a candidate;
 * init_sliced (nullable): the caller's sliced set, kept as a candidate plan.
 * out_children: (n-1)*2 ints; out_sliced: capacity n_index, pick order
 * (the engine's MSB-first mask order, engine.py:276-279).
 * out_stats[8]: log2 cost per slice, max rank, log2 total, log2 best
 * unsliced candidate, candidate trees, seconds, winning plan, plans tried.
 * Returns 0, 1 (bad input), 2 (target unreachable), 3 (internal error);
 * tnbp_last_error() describes the failure. */
int tnbp_optimize(int n_leaves, const int* leaf_ptr, const int* leaf_idx, int n_index,
                  const unsigned char* sliceable, const int* init_children,
                  const int* init_sliced, int n_init_sliced, const tnbp_options* opt,
                  int* out_children, int* out_sliced, int* out_n_sliced, double* out_stats);

/* Cost of a given tree + sliced set under objective 0/1:
 * out_stats[3] = {log2 cost per slice, max rank, log2 total}. */
int tnbp_tree_cost(int n_leaves, const int* leaf_ptr, const int* leaf_idx, int n_index,
                   const int* children, const int* sliced, int n_sliced, int objective,
                   double* out_stats);

/* Pairwise order of a whole (small) network, no slicing: a deterministic
 * size-reduction greedy, then every subtree of <= opt->polish_k operands
 * re-optimised exactly under opt->objective (the whole order when
 * n_leaves <= polish_k), intermediates kept <= max(opt->target_log2, the
 * greedy's largest).  Used for the head-absorbed tail (the reference orders
 * its tail with the greedy of ordering.py:256-285 and contracts it per
 * pinned block, engine.py:348-377).  Open legs (one endpoint) stay open.
 * out_children: (n-1)*2 ints, SSA post-order as in tnbp_optimize.
 * out_stats[3] = {log2 model cost, max rank, log2 multiplications}. */
int tnbp_order(int n_leaves, const int* leaf_ptr, const int* leaf_idx, int n_index,
               const tnbp_options* opt, int* out_children, double* out_stats);

const char* tnbp_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* TNB_PLAN_H */
