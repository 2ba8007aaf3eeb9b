// Program = compiled pairwise contraction schedule + device buffers.
//
// Host-side compilation (once per (network topology, tree, slicing)):
//   * axis lists for every leaf (sliced axes removed) and step result,
//     exactly the index bookkeeping of tncut `_contract_steps`
//     (engine.py:117-144): shared = a_ids & b_ids in a's order, result =
//     free axes of the two operands;
//   * slice dependence: a tensor is slice-variant iff some leaf below it
//     carries a sliced index; invariant subtrees are computed once and kept
//     (hoisting) -- they do not change with the mask;
//   * per step a kernel choice (tcgen05 3xFP16 GEMM or SIMT), the
//     canonical-layout byte LUTs, and -- for the tensor-core path -- the
//     operand roles (smaller operand is expanded) and TMA descriptors;
//   * a first-fit arena for slice-variant intermediates (liveness in step
//     order) that also holds each tensor-core step's operand staging for the
//     duration of that step.
// Execution of a slice range follows compute_head_vector's loop
// (engine.py:275-298) with the binary-counter fixed-mode sum
// (engine.py:207-222) or the free running sum.
#include "tnb_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <unordered_map>

namespace tnb {

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

namespace {

constexpr int64_t kAlign = 1024;
inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int ilog2(int64_t x) {
  int l = 0;
  while (((int64_t)1 << l) < x) ++l;
  return l;
}

struct Arena {
  // first-fit allocator over a virtual offset space
  std::map<int64_t, int64_t> free_;  // offset -> size
  int64_t top = 0;
  int64_t alloc(int64_t size) {
    size = align_up(size, kAlign);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second >= size) {
        const int64_t off = it->first;
        const int64_t rest = it->second - size;
        free_.erase(it);
        if (rest > 0) free_[off + size] = rest;
        return off;
      }
    }
    // extend: merge with a trailing free block if there is one
    if (!free_.empty()) {
      auto last = std::prev(free_.end());
      if (last->first + last->second == top) {
        const int64_t off = last->first;
        free_.erase(last);
        top = off + size;
        return off;
      }
    }
    const int64_t off = top;
    top += size;
    return off;
  }
  void release(int64_t off, int64_t size) {
    size = align_up(size, kAlign);
    auto it = free_.emplace(off, size).first;
    // coalesce with next
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }
};

enum Pool { POOL_LEAF = 0, POOL_SLICE = 1, POOL_PERSIST = 2, POOL_ARENA = 3 };

struct TensorRec {
  std::vector<int64_t> axes;
  bool variant = false;
  uint64_t dep = 0;     // mask bits this tensor depends on (reuse mode)
  bool cached = false;  // reuse mode: value must survive across masks (dedicated buffer)
  int pool = POOL_LEAF;
  int64_t off = 0;  // element offset within the pool
  int64_t elems = 1;
  int leaf_pos = -1;
  int def_step = -1;   // step producing it (-1: leaf)
  int last_use = -1;   // last consuming step (n_steps: the root)
  int fuse_role = 0;   // 1/2: stored as its consumer's staged rows/cols operand (fp16 hi/lo)
};

enum StepKind { KIND_SIMT = 0, KIND_TC = 1 };

struct StepRec {
  int a = -1, b = -1, out = -1;
  int kind = KIND_SIMT;
  bool hoisted = false;
  bool has_key = false;   // reuse mode: output valid for mask bits `last_key`
  uint64_t last_key = 0;
  int64_t M = 1, N = 1, K = 1;   // SIMT: rows of a, cols of b, shared. TC: rows/cols operand.
  int rows_t = -1, cols_t = -1;  // TC operand tensors (rows unexpanded, cols expanded)
  int lut_a = -1, lut_b = -1;    // SIMT: indices into the LUT table
  int lut_e = -1;                // small-K SIMT: output-quad enumeration LUT (-1: identity)
  std::vector<int> canon_rows, canon_cols;  // TC: canonical bit -> source bit
  int st_rows = -1, st_cols = -1;           // TC: indices into Program::stages
  double mults = 0;
  int64_t scratch_off = 0, scratch_bytes = 0;  // TC: staging region in the arena (bytes)
  bool fuse_rows = false, fuse_cols = false;   // TC: operand written by its producer's epilogue
  int fuse_consumer = -1;                      // step whose operand this step's output is written as
  FuseOut simt_fuse;                           // SIMT (small-K) producer: fused output map
  int batch = -1;                              // tiled SIMT step launched in Program::batches[batch]
  TcGemmPlan tc;
  // fp16 scale guard of a fused producer: right after it, the re-run launch
  // (tc_redo / simt_redo, FuseOut::redo) compares the a-priori bound it scaled
  // by with its result's exact max; if the bound is more than
  // Program::guard_bits binary orders looser it rewrites the operand scaled
  // by the exact max, else exits at once.  The decision lands in *guard,
  // which the consumer's ScaleSrc follows
  bool dstage = false;  // fp64 wide step: operands permuted to [M][K] / [N][K] first (scratch)
  bool has_redo = false;
  unsigned int* guard = nullptr;
  TcGemmPlan tc_redo;
  FuseOut simt_redo;
};

// bytes of a tensor's storage: complex elements, or the consumer's fp16
// hi/lo planes when its producer's epilogue writes it in staged form
inline int64_t tensor_bytes(const TensorRec& t, int64_t esize) {
  if (t.fuse_role == 1) return 8 * t.elems;
  if (t.fuse_role == 2) return 16 * t.elems;
  return esize * t.elems;
}

}  // namespace

// ---------------------------------------------------------------------------
struct Program {
  int device = 0;
  int precision = TNB_SINGLE;
  uint32_t flags = 0;
  size_t esize = 8;  // bytes per complex element
  int num_sms = 148;
  cudaStream_t stream = nullptr;

  int n_sliced = 0;
  std::vector<TensorRec> tensors;        // leaves first (leaf_pos order), then step outputs
  std::vector<StepRec> steps;
  std::vector<int32_t> leaf_ranks;
  std::vector<int64_t> leaf_pool_off;    // element offset of full leaf data in the leaf pool
  std::vector<ByteLut> luts;
  int root = -1;
  int root_lut = -1;
  int64_t out_elems = 1;
  bool root_identity = false;

  // device memory
  void* d_leaf_pool = nullptr;   int64_t leaf_pool_elems = 0;
  void* d_slice_pool = nullptr;  int64_t slice_pool_elems = 0;
  void* d_persist = nullptr;     int64_t persist_elems = 0;
  void* d_arena = nullptr;       int64_t arena_bytes = 0;
  int64_t scratch_bytes = 0;     // largest per-step staging region (inside the arena)
  ByteLut* d_luts = nullptr;
  SlicedLeafDesc* d_sl_descs = nullptr; int n_sl_descs = 0;
  uint32_t* d_keep = nullptr;
  unsigned int* d_tmax = nullptr;   // per-tensor max|re|,|im| slots (fp32 bits)
  unsigned int* d_progress = nullptr;  // GEMM soft-pacing counters (one per CTA unit)
  unsigned int* d_guard = nullptr;  // fp16 scale guard words (per tensor slot) + redo counter
  int guard_bits = 18;              // TNB_SCALE_GUARD_BITS at creation (< 0: guard off)
  int lut_ident = -1;               // identity LUT (staged fp64 operands are canonical)
  std::vector<int> slot;            // tensor -> slot
  int inv_slot_begin = 0, inv_slot_count = 0, var_slot_begin = 0, var_slot_count = 0;
  std::vector<StageTables> stages;  // device views of the TC staging tables
  uint32_t* d_stage_u32 = nullptr;
  ByteLut* d_stage_luts = nullptr;
  ByteLut* d_fuse_luts = nullptr;   // fused-staging destination maps (2 per fused edge)
  struct SimtBatch { int first_step, last_step, n; int64_t blocks; SimtStepDesc* d_descs; };
  std::vector<SimtBatch> batches;   // independent consecutive tiled-SIMT steps, one launch each
  SimtStepDesc* d_simt_descs = nullptr;
  // per-slice launch plan as CUDA-graph segments: the runs of small kernels
  // between GEMMs are captured once and replayed per mask; GEMMs stay direct
  // launches (their CUDA-event timing feeds the roofline figures)
  struct Segment { cudaGraphExec_t exec = nullptr; int kernels = 0; };
  struct PlanItem { int seg = -1, step = -1; };
  std::vector<Segment> segs;
  std::vector<PlanItem> items;
  bool segs_built = false;
  int n_fused = 0;
  void* d_acc = nullptr;          // (n_sliced + 2) accumulator slots of out_elems
  int n_acc_slots = 0;
  bool invariant_valid = false;
  bool reuse = false;               // TNB_FLAG_REUSE_SLICES
  int64_t reuse_bytes = 0;          // dedicated buffers of cross-slice cached tensors

  // timing
  int timing = 0;                   // 0 off, 1 all kernel classes, 2 GEMM + total
  tnb_timing last{};
  std::vector<cudaEvent_t> ev_pool;

  // stats
  double flops_per_slice = 0, tc_flops_per_slice = 0;
  int n_tc = 0, n_simt = 0, n_hoisted = 0;

  ~Program() {
    if (device >= 0) cudaSetDevice(device);
    void* ptrs[] = {d_leaf_pool, d_slice_pool, d_persist, d_arena, d_luts,
                    d_sl_descs, d_keep, d_tmax, d_acc, d_stage_u32, d_stage_luts, d_progress, d_fuse_luts, d_simt_descs,
                    d_guard};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& g : segs) if (g.exec) cudaGraphExecDestroy(g.exec);
    if (stream) cudaStreamDestroy(stream);
  }

  void* tensor_ptr(int t) const {
    const TensorRec& r = tensors[t];
    char* base = nullptr;
    switch (r.pool) {
      case POOL_LEAF: base = (char*)d_leaf_pool; break;
      case POOL_SLICE: base = (char*)d_slice_pool; break;
      case POOL_PERSIST: base = (char*)d_persist; break;
      default: base = (char*)d_arena; break;
    }
    return base + (size_t)r.off * esize;
  }
};

namespace {

// canonical (row, k) index -> source element offset in tensor `t`:
// canonical bit p < nk <-> kaxes[nk-1-p]; bit p >= nk <-> raxes[nr-1-(p-nk)].
std::vector<int> canon_bits(const std::vector<int64_t>& axes, const std::vector<int64_t>& raxes,
                            const std::vector<int64_t>& kaxes) {
  const int r = (int)axes.size();
  std::unordered_map<int64_t, int> pos;
  for (int i = 0; i < r; ++i) pos[axes[i]] = i;
  std::vector<int> src;
  src.reserve(r);
  for (int p = 0; p < (int)kaxes.size(); ++p) src.push_back(r - 1 - pos.at(kaxes[kaxes.size() - 1 - p]));
  for (int p = 0; p < (int)raxes.size(); ++p) src.push_back(r - 1 - pos.at(raxes[raxes.size() - 1 - p]));
  return src;
}

// Enumeration order of the small-K kernel's output quads (4 consecutive
// columns per thread): thread-index bit p -> output-quad bit order[p].
// Lane bits 0-4 stay on the output's lowest quad bits (the store pattern the
// fusion planner arranged); the next bits are the output bits holding the
// big operand's lowest storage bits, so a 2^11-quad window of threads reads
// whole lines of it (before: a fused producer's planned orders could put
// those bits 2^20 threads apart, and every 8-B gather cost a DRAM line).
// src_x: canonical bit -> storage bit (canon_bits: k bits first, then free).
std::vector<int> smallk_enumeration(const std::vector<int>& src_a, const std::vector<int>& src_b,
                                    int lm, int ln, int lk, int mode) {
  const int Q = lm + ln - 2;
  std::vector<int> order;
  std::vector<char> used(std::max(Q, 0), 0);
  const bool a_big = lm >= ln;
  const std::vector<int>& src = a_big ? src_a : src_b;
  std::vector<int> inv(src.size(), -1);
  for (int c = 0; c < (int)src.size(); ++c) inv[src[c]] = c;
  int sb = 0;
  auto place_src = [&](int count) {  // next `count` output-quad bits by source storage order
    int placed = 0;
    for (; sb < (int)inv.size() && placed < count; ++sb) {
      const int c = inv[sb];
      if (c < lk) continue;                          // contracted: every thread loops over k
      const int ob = a_big ? ln + (c - lk) : c - lk;  // output bit (n bits lowest)
      if (ob < 2) continue;                          // per-thread vector bits
      const int qb = ob - 2;
      if (qb >= Q || used[qb]) continue;
      order.push_back(qb);
      used[qb] = 1;
      ++placed;
    }
  };
  auto place_out = [&](int count) {
    for (int j = 0, placed = 0; j < Q && placed < count; ++j)
      if (!used[j]) { order.push_back(j); used[j] = 1; ++placed; }
  };
  if (mode == 3) {
    // auto: keep the output on the lanes when the big operand's lowest
    // storage bits (below the per-thread/contracted ones) already map there
    std::vector<char> lane(std::max(Q, 0), 0);
    for (int j = 0; j < std::min(5, Q); ++j) lane[j] = 1;
    int seen = 0, on_lanes = 0;
    for (int b = 0; b < (int)inv.size() && seen < 3; ++b) {
      const int c = inv[b];
      if (c < lk) continue;
      const int ob = a_big ? ln + (c - lk) : c - lk;
      if (ob < 2 || ob - 2 >= Q) continue;
      ++seen;
      on_lanes += lane[ob - 2];
    }
    mode = seen > 0 && on_lanes == seen ? 1 : 2;
  }
  if (mode == 2) {  // lanes read the big operand's lines; output runs right above
    place_src(5);
    place_out(6);
  } else {          // lanes write the output's lines; source lines right above
    place_out(5);
    place_src(6);
  }
  for (int qb = 0; qb < Q; ++qb)
    if (!used[qb]) order.push_back(qb);
  return order;
}

int add_lut(Program* P, const std::vector<int>& src_bit) {
  ByteLut l;
  build_lut(src_bit, &l);
  P->luts.push_back(l);
  return (int)P->luts.size() - 1;
}

// parts of a step's launches: SIMT kernels / operand staging (kPre), the
// tensor-core GEMM (kGemm), the split-K reduce (kPost)
enum StepPart { kPre = 1, kGemm = 2, kPost = 4, kAll = 7 };

template <typename T>
void exec_step(Program* P, StepRec& s, int parts = kAll);

template <typename T>
void build_segments(Program* P);

template <typename T>
void run_range_t(Program* P, uint64_t a, uint64_t b, int mode, void* out, bool out_dev);

}  // namespace

void upload_leaf_max(Program* P, int leaf_pos, const double* data);

// ---------------------------------------------------------------------------
// SIMT batching (program_create): fills P->batches and StepRec::batch.
void plan_simt_batches(Program* P) {
  const int n_steps = (int)P->steps.size();
  // SIMT batching: consecutive tiled-SIMT steps of one execution
  // sequence (the hoisted pass, or the per-slice pass) that do not consume
  // each other's results run as one launch.  Memory planning below keeps
  // every operand of a batch live until its last member, so members never
  // alias each other's inputs or outputs.
  {
    static const int batch_env = env_int("TNB_SIMT_BATCH", 1);
    const bool batching = batch_env && !P->reuse;
    for (int seq = 0; batching && seq < 2; ++seq) {
      std::vector<int> cur;
      auto close = [&] {
        if (cur.size() >= 2) {
          Program::SimtBatch b{cur.front(), cur.back(), (int)cur.size(), 0, nullptr};
          for (int i : cur) P->steps[i].batch = (int)P->batches.size();
          P->batches.push_back(b);
        }
        cur.clear();
      };
      for (int i = 0; i < n_steps; ++i) {
        StepRec& s = P->steps[i];
        if ((int)s.hoisted != seq) continue;  // seq 1: hoisted pass, seq 0: per slice
        const bool cand = s.kind == KIND_SIMT && !simt_uses_smallk(s.M, s.N, s.K) &&
                          !simt_uses_wide(s.M, s.N, s.K) && P->tensors[s.out].fuse_role == 0;
        if (!cand) { close(); continue; }
        bool dep = false;
        for (int m : cur)
          if (P->steps[m].out == s.a || P->steps[m].out == s.b) dep = true;
        if (dep || cur.size() >= 128) close();
        cur.push_back(i);
      }
      close();
    }
  }
}

// Memory planning (program_create): pools, arena offsets and per-step
// staging scratch; releases of a SIMT batch's operands wait for its last member.
void plan_memory(Program* P) {
  const int n_steps = (int)P->steps.size();
  std::vector<int> batch_last(n_steps, -1);  // step -> global index of its batch's last member
  for (auto& b : P->batches)
    for (int i = b.first_step; i <= b.last_step; ++i)
      if (P->steps[i].batch >= 0 && &P->batches[P->steps[i].batch] == &b) batch_last[i] = b.last_step;

  // memory planning: persistent (hoisted) and arena (variant) tensors
  int64_t persist_off = 0;
  Arena arena;
  std::vector<std::vector<int>> free_after(n_steps + 1);
  for (int t = 0; t < (int)P->tensors.size(); ++t) {
    const TensorRec& r = P->tensors[t];
    if (r.def_step >= 0 && r.last_use >= 0 && r.last_use < n_steps) free_after[r.last_use].push_back(t);
  }
  int64_t scratch_bytes = 0;
  static const int dstage_env = env_int("TNB_DSTAGE", 1);
  std::vector<std::vector<int>> deferred(n_steps + 1);
  for (int i = 0; i < n_steps; ++i) {
    StepRec& s = P->steps[i];
    TensorRec& o = P->tensors[s.out];
    const int64_t ob = tensor_bytes(o, (int64_t)P->esize);  // fused: the consumer's fp16 planes
    if (s.hoisted || !o.variant || o.cached) {
      o.pool = POOL_PERSIST;
      o.off = persist_off;
      persist_off += align_up(ob / (int64_t)P->esize, 128);
      if (o.cached) P->reuse_bytes += ob;
    } else {
      o.pool = POOL_ARENA;
      o.off = arena.alloc(ob) / (int64_t)P->esize;
    }
    if (s.kind == KIND_SIMT && s.batch < 0 && P->precision == TNB_DOUBLE && dstage_env &&
        simt_uses_wide(s.M, s.N, s.K)) {
      // fp64 wide step: both operands permuted once into canonical row-major
      // [M][K] / [N][K] (the tile loads are then coalesced instead of gathered
      // N/64 resp. M/64 times); scratch for this step only, like TC staging
      s.dstage = true;
      const int64_t need = align_up(s.M * s.K * 16, kAlign) + s.N * s.K * 16;
      s.scratch_bytes = need;
      s.scratch_off = arena.alloc(need);
      scratch_bytes = std::max(scratch_bytes, need);
      if (P->lut_ident < 0) {
        std::vector<int> ident(32);
        for (int b = 0; b < 32; ++b) ident[b] = b;
        P->lut_ident = add_lut(P, ident);
      }
    }
    if (s.kind == KIND_TC) {
      // operand staging (+ split-K workspace) lives in the arena for the
      // duration of this step only: it shares memory with dead tensors.
      // Fused operands are already staged (their producer wrote them).
      const int64_t Kp = 2 * s.K, Np = 2 * s.N;
      int64_t need = (s.fuse_rows ? 0 : 2 * s.M * Kp * 2) + (s.fuse_cols ? 0 : 2 * Np * Kp * 2);
      need = align_up(need, kAlign) + tc_workspace_elems(s.M, Np, Kp, P->num_sms) * 4;
      s.scratch_bytes = need;
      if (need > 0) s.scratch_off = arena.alloc(need);
      scratch_bytes = std::max(scratch_bytes, need);
    }
    // variant operands whose last use is this step are released after it
    // (after the batch's last member when the step runs in a SIMT batch)
    const int rel_at = batch_last[i] >= 0 ? batch_last[i] : i;
    if (rel_at != i) {
      deferred[rel_at].insert(deferred[rel_at].end(), free_after[i].begin(), free_after[i].end());
    } else {
      for (int t : free_after[i]) {
        TensorRec& r = P->tensors[t];
        if (r.pool == POOL_ARENA) arena.release(r.off * (int64_t)P->esize, tensor_bytes(r, (int64_t)P->esize));
      }
    }
    for (int t : deferred[i]) {
      TensorRec& r = P->tensors[t];
      if (r.pool == POOL_ARENA) arena.release(r.off * (int64_t)P->esize, tensor_bytes(r, (int64_t)P->esize));
    }
    if ((s.kind == KIND_TC || s.dstage) && s.scratch_bytes > 0) arena.release(s.scratch_off, s.scratch_bytes);
  }
  P->persist_elems = persist_off;
  P->arena_bytes = arena.top;
  P->scratch_bytes = scratch_bytes;

}

// ---------------------------------------------------------------------------
// Tensor-core plans (program_create): TMA descriptors over the fixed operand
// addresses, the fp16 scale source of every operand, and the fused-staging
// destination maps (GEMM epilogues and small-K SIMT producers).
void plan_tensor_core_steps(Program* P) {
  const int n_steps = (int)P->steps.size();
  auto dmalloc = [](void** p, int64_t bytes) {
    if (bytes <= 0) bytes = 256;
    TNB_CUDA(cudaMalloc(p, (size_t)bytes));
  };
  dmalloc((void**)&P->d_progress, (int64_t)P->num_sms * 4);
  // fp16 split scale of a tensor-core operand: its own max when staged, the
  // producer's a-priori bound 2 K max|A| max|B| when the producer's epilogue
  // wrote it (fused); producer and consumer evaluate the same ScaleSrc
  {
    const char* e = getenv("TNB_SCALE_GUARD_BITS");
    P->guard_bits = e ? atoi(e) : 18;
  }
  // producer view (the bound alone) and consumer view (bound, or the
  // result's exact max when the guard fired) of a fused operand's scale
  auto bound_scale = [&](int t) {
    ScaleSrc sc;
    const TensorRec& r = P->tensors[t];
    if (r.fuse_role != 0) {
      const StepRec& p = P->steps[r.def_step];
      sc.a = P->d_tmax + P->slot[p.kind == KIND_TC ? p.rows_t : p.a];
      sc.b = P->d_tmax + P->slot[p.kind == KIND_TC ? p.cols_t : p.b];
      sc.f = (float)(2.0 * (double)p.K);
    } else {
      sc.a = P->d_tmax + P->slot[t];
    }
    return sc;
  };
  auto operand_scale = [&](int t) {
    ScaleSrc sc = bound_scale(t);
    if (P->tensors[t].fuse_role != 0 && P->guard_bits >= 0) {
      sc.guard = P->d_guard + P->slot[t];
      sc.own = P->d_tmax + P->slot[t];
    }
    return sc;
  };
  std::vector<ByteLut> fuse_luts;
  std::vector<int> fuse_lut_step;
  // destination map of a fused result in its consumer's operand layout
  // (stage_kernel's): canonical (row r, k) -> half2 index (k >> L, r,
  // k & (2^L-1)) in [K/2^L][rows][2^L], a zero bit inserted at L for the
  // expanded cols operand.  Returns the destination bit of every result
  // column bit (nvec) and row bit (mvec); fills everything but the kernel-
  // specific store-path fields.
  auto build_fuse_map = [&](int i, StepRec& s, FuseOut& f, std::vector<int>& nvec, std::vector<int>& mvec) {
    const TensorRec& o = P->tensors[s.out];
    const StepRec& c = P->steps[s.fuse_consumer];
    const bool as_rows = o.fuse_role == 1;
    const std::vector<int>& canon = as_rows ? c.canon_rows : c.canon_cols;
    const int nk = ilog2(c.K), nr = ilog2(as_rows ? c.M : c.N);
    const int L = std::min(nk, kKBlockLog);
    const int nbits = (int)o.axes.size();
    if (nbits != nk + nr || (int)canon.size() != nbits) throw Error(TNB_ERR_SHAPE, "fused staging: rank mismatch");
    std::vector<int> dbit(nbits);
    for (int p = 0; p < nbits; ++p) {
      int db = p < L ? p : (p < nk ? p + nr : p - nk + L);
      if (!as_rows && db >= L) db += 1;
      dbit[canon[p]] = db;
    }
    const int ln = ilog2(s.N);  // result columns = the low source bits
    nvec.assign(dbit.begin(), dbit.begin() + ln);
    mvec.assign(dbit.begin() + ln, dbit.end());
    f.mode = as_rows ? 1 : 2;
    f.L = L;
    for (int j = 0; j < 32; ++j) {
      uint32_t v = 0;
      for (int p = 0; p < std::min(5, ln); ++p)
        if ((j >> p) & 1) v |= 1u << nvec[p];
      f.dlow[j] = v;
    }
    f.hi = (__half2*)P->tensor_ptr(s.out);
    f.lo = f.hi + (as_rows ? c.M * c.K : 2 * c.N * c.K);
    f.scale = bound_scale(s.out);  // the producer's first run scales by the bound
    fuse_luts.emplace_back();
    build_lut(mvec, &fuse_luts.back());
    fuse_luts.emplace_back();
    build_lut(nvec, &fuse_luts.back());
    fuse_lut_step.push_back(i);
  };
  auto debug_fuse = [&](int i, const StepRec& s, const FuseOut& f, const std::vector<int>& nvec,
                        const std::vector<int>& mvec) {
    if (!getenv("TNB_DEBUG_FUSE")) return;
    fprintf(stderr, "TNB_FUSE step %d (%s) -> %d role %d out 2^%d fast %d vec %d nvec[0..4]", i,
            s.kind == KIND_TC ? "tc" : "smallk", s.fuse_consumer, f.mode, (int)(nvec.size() + mvec.size()),
            f.fast, f.vec);
    for (size_t p = 0; p < std::min<size_t>(5, nvec.size()); ++p) fprintf(stderr, " %d", nvec[p]);
    fprintf(stderr, " mvec[0..4]");
    for (size_t p = 0; p < std::min<size_t>(5, mvec.size()); ++p) fprintf(stderr, " %d", mvec[p]);
    fprintf(stderr, " lane_w");
    for (int b = 0; b < 5; ++b) fprintf(stderr, " %d", f.fast ? ilog2(f.lane_w[b]) : -1);
    fprintf(stderr, " exchanges %d\n", (f.xlane[0] != 0) + (f.xlane[1] != 0) + (f.xlane[2] != 0));
  };
  for (int i = 0; i < n_steps; ++i) {
    StepRec& s = P->steps[i];
    std::vector<int> nvec, mvec;
    if (s.kind != KIND_TC) {
      if (P->tensors[s.out].fuse_role == 0) continue;
      // fused small-K SIMT producer: a thread owns 4 consecutive columns
      if (!simt_uses_smallk(s.M, s.N, s.K)) throw Error(TNB_ERR_SHAPE, "fused output on a tiled SIMT step");
      build_fuse_map(i, s, s.simt_fuse, nvec, mvec);
      s.simt_fuse.vec = nvec.size() >= 2 && nvec[0] == 0 && nvec[1] == 1;
      debug_fuse(i, s, s.simt_fuse, nvec, mvec);
      continue;
    }
    const int64_t Kp = 2 * s.K, Np = 2 * s.N;
    char* base = (char*)P->d_arena + s.scratch_off;
    int64_t used = 0;
    __half* ahi = s.fuse_rows ? (__half*)P->tensor_ptr(s.rows_t) : (__half*)base;
    if (!s.fuse_rows) used += 2 * s.M * Kp * 2;
    __half* alo = ahi + s.M * Kp;
    __half* bhi = s.fuse_cols ? (__half*)P->tensor_ptr(s.cols_t) : (__half*)(base + used);
    if (!s.fuse_cols) used += 2 * Np * Kp * 2;
    __half* blo = bhi + Np * Kp;
    float* ws = (float*)(base + align_up(used, kAlign));
    const int64_t ws_elems = tc_workspace_elems(s.M, Np, Kp, P->num_sms);
    tc_plan_gemm(&s.tc, ahi, alo, bhi, blo, s.M, Np, Kp, (float*)P->tensor_ptr(s.out), ws, ws_elems,
                 operand_scale(s.rows_t), operand_scale(s.cols_t), P->d_tmax + P->slot[s.out],
                 P->num_sms);
    s.tc.progress = P->d_progress;
    if (getenv("TNB_DEBUG_GEMM"))
      fprintf(stderr, "TNB_GEMM step %d M %lld Np %lld Kp %lld cg %d nb %d splits %d fused_out %d rows_fused %d cols_fused %d hoisted %d grid %d skinny %d\n",
              i, (long long)s.M, (long long)Np, (long long)Kp, s.tc.cta_group, s.tc.nb, s.tc.splits,
              P->tensors[s.out].fuse_role, (int)s.fuse_rows, (int)s.fuse_cols, (int)s.hoisted, s.tc.grid,
              s.tc.skinny);
    if (P->tensors[s.out].fuse_role == 0) continue;
    if (s.tc.splits != 1) throw Error(TNB_ERR_SHAPE, "fused staging planned for a split-K step");
    FuseOut& f = s.tc.fuse;
    build_fuse_map(i, s, f, nvec, mvec);
    const int ln = (int)nvec.size();
    // fast path: vector bits n0,n1 -> destination bits 0,1; the lanes take
    // the 5 thread-local source bits (slot bits n2..n(1+sb), lane bits
    // m0..m4) with the lowest destination bits, swapped in by butterfly
    // exchanges.  sb = 3 slot bits (32 complex per thread); sb = 2 for
    // 16-column results (narrow consumers' operands)
    f.fast = 0;
    static const int fast_env = env_int("TNB_FUSE_FAST", 1);
    if (fast_env && ln >= 4 && (int)mvec.size() >= 5 && nvec[0] == 0 && nvec[1] == 1) {
      const int sb = std::min(3, ln - 2);
      std::vector<std::pair<int, int>> loc;  // (destination bit, local bit: 0..sb-1 slot, sb.. lane)
      for (int j = 0; j < sb; ++j) loc.push_back({nvec[2 + j], j});
      for (int b = 0; b < 5; ++b) loc.push_back({mvec[b], sb + b});
      std::sort(loc.begin(), loc.end());
      std::vector<char> on_lane(sb + 5, 0);
      for (int x = 0; x < 5; ++x) on_lane[loc[x].second] = 1;
      int dslot[3] = {0, 0, 0}, dlane[5];
      for (int j = 0; j < sb; ++j) dslot[j] = nvec[2 + j];
      for (int b = 0; b < 5; ++b) dlane[b] = mvec[b];
      int b = 0;
      for (int j = 0; j < 3; ++j) {
        f.xlane[j] = 0;
        if (j >= sb || !on_lane[j]) continue;   // slot bit stays in the registers
        while (on_lane[sb + b]) ++b;            // a lane bit that must leave the lanes
        f.xlane[j] = 1 << b;
        std::swap(dslot[j], dlane[b]);
        ++b;
      }
      for (int bb = 0; bb < 5; ++bb) f.lane_w[bb] = 1u << dlane[bb];
      for (int q = 0; q < 8; ++q) {
        uint32_t v = 0;
        for (int j = 0; j < sb; ++j)
          if ((q >> j) & 1) v |= 1u << dslot[j];
        f.slot_w[q] = v;
      }
      f.nslot = 1 << sb;
      f.fast = 1;
    }
    debug_fuse(i, s, f, nvec, mvec);
  }
  P->n_fused = (int)fuse_lut_step.size();
  if (!fuse_luts.empty()) {
    dmalloc((void**)&P->d_fuse_luts, (int64_t)fuse_luts.size() * sizeof(ByteLut));
    TNB_CUDA(cudaMemcpy(P->d_fuse_luts, fuse_luts.data(), fuse_luts.size() * sizeof(ByteLut),
                        cudaMemcpyHostToDevice));
    for (size_t e = 0; e < fuse_lut_step.size(); ++e) {
      StepRec& st = P->steps[fuse_lut_step[e]];
      FuseOut& f = st.kind == KIND_TC ? st.tc.fuse : st.simt_fuse;
      f.lut_m = P->d_fuse_luts + 2 * e;
      f.lut_n = P->d_fuse_luts + 2 * e + 1;
    }
  }
  // scale-guard re-runs of every fused producer: the same launch again; its
  // prologue decides (bound vs the result's exact max) whether to rewrite the
  // operand scaled by the exact max, records that in the guard word the
  // consumer's ScaleSrc reads, and otherwise exits at once
  if (P->guard_bits >= 0) {
    for (int i = 0; i < n_steps; ++i) {
      StepRec& st = P->steps[i];
      FuseOut& f = st.kind == KIND_TC ? st.tc.fuse : st.simt_fuse;
      if (f.mode == 0) continue;
      st.has_redo = true;
      st.guard = P->d_guard + P->slot[st.out];
      FuseOut r = f;
      r.redo = 1;
      r.guard_bits = P->guard_bits;
      r.guard_bound = f.scale;
      r.guard_word = st.guard;
      r.guard_count = P->d_guard + P->slot.size();
      r.scale = ScaleSrc{};
      r.scale.a = P->d_tmax + P->slot[st.out];
      if (st.kind == KIND_TC) {
        st.tc_redo = st.tc;
        st.tc_redo.fuse = r;
      } else {
        st.simt_redo = r;
      }
    }
  }

}

// ---------------------------------------------------------------------------
// Index-order planning (the pre-pass of program_create).
// Pre-pass over index sets: kernel kind and operand roles of every
// step, the fused-staging edges (a tensor-core step whose result feeds a
// tensor-core step writes it in the consumer's staged fp16 layout from its
// epilogue), and the canonical index orders of every tensor-core step.
// Orders are planned consumer-first (reverse step order): a consumer puts
// contracted indices that sit on its producer's lowest result columns on
// its lowest K bits, and the producer then orders its free indices so that
// the consumer's lowest destination bits (low K bits, then the consumer's
// lowest free bits) are its thread-local columns / lane-local rows -- the
// epilogue's scattered stores then form contiguous runs.  Lists below are
// lowest-first (canonical bit 0 first).
struct OrderPlan {
  std::vector<std::vector<int64_t>> ord_k, ord_rows, ord_cols;  // per step, lowest-first
  std::vector<char> rows_is_a;      // SIMT small-K producer: m/n roles swapped if 0
  std::vector<int> fuse_role;       // tensor -> 1/2 when written as its consumer's operand
  std::vector<int> fuse_consumer;   // tensor -> consuming step
};

template <typename Eligible>
OrderPlan plan_orders(const tnb_program_desc* d, const Program* P, bool use_tc, const Eligible& tc_eligible) {
  OrderPlan op;
  op.ord_k.resize(d->n_steps);
  op.ord_rows.resize(d->n_steps);
  op.ord_cols.resize(d->n_steps);
  op.rows_is_a.assign(d->n_steps, 1);
  auto& ord_k = op.ord_k;
  auto& ord_rows = op.ord_rows;
  auto& ord_cols = op.ord_cols;
  auto& pre_rows_is_a = op.rows_is_a;
  auto& fuse_role_pre = op.fuse_role;
  auto& fuse_consumer_pre = op.fuse_consumer;
  {
    static const int fuse_env = [] {
      const char* e = getenv("TNB_FUSE");
      return e ? atoi(e) : 1;
    }();
    const int nt = d->n_leaves + d->n_steps;
    std::vector<std::vector<int64_t>> sets(nt);
    std::vector<int> def(nt, -1);
    for (int i = 0; i < d->n_leaves; ++i) sets[i] = P->tensors[i].axes;
    std::unordered_map<int64_t, int> ids;
    for (int i = 0; i < d->n_leaves; ++i) ids[d->leaf_ids[i]] = i;
    // rows/cols: the GEMM's M/N sides (tensor-core steps: rows = larger
    // operand's free indices; SIMT steps: rows = a's, cols = b's, the m/n of
    // the SIMT kernels).  smallk: a SIMT step on the streaming small-K kernel
    // (launch_contract_simt), whose result may also be written fused.
    struct Pre { int a = -1, b = -1; bool tc = false, smallk = false, rows_is_a = true; std::vector<int64_t> shared, rows, cols; };
    std::vector<Pre> pre(d->n_steps);
    for (int i = 0; i < d->n_steps; ++i) {
      auto ia = ids.find(d->steps[3 * i]), ib = ids.find(d->steps[3 * i + 1]);
      if (ia == ids.end() || ib == ids.end() || d->steps[3 * i] == d->steps[3 * i + 1])
        throw Error(TNB_ERR_SHAPE, "step " + std::to_string(i) + " references a missing operand");
      Pre& q = pre[i];
      q.a = ia->second;
      q.b = ib->second;
      ids.erase(ia);
      ids.erase(ids.find(d->steps[3 * i + 1]));
      const auto& A = sets[q.a];
      const auto& B = sets[q.b];
      std::vector<int64_t> afree, bfree;
      for (int64_t x : A) (std::find(B.begin(), B.end(), x) != B.end() ? q.shared : afree).push_back(x);
      for (int64_t x : B) if (std::find(A.begin(), A.end(), x) == A.end()) bfree.push_back(x);
      const int na = (int)afree.size(), nb = (int)bfree.size(), nab = (int)q.shared.size();
      q.tc = tc_eligible(na, nb, nab);
      q.rows_is_a = q.tc ? na >= nb : true;
      q.smallk = use_tc && !q.tc && simt_uses_smallk((int64_t)1 << na, (int64_t)1 << nb, (int64_t)1 << nab);
      q.rows = q.rows_is_a ? afree : bfree;
      q.cols = q.rows_is_a ? bfree : afree;
      ord_k[i].assign(q.shared.rbegin(), q.shared.rend());
      ord_rows[i].assign(q.rows.rbegin(), q.rows.rend());
      ord_cols[i].assign(q.cols.rbegin(), q.cols.rend());
      const int out = d->n_leaves + i;
      sets[out] = afree;
      sets[out].insert(sets[out].end(), bfree.begin(), bfree.end());
      def[out] = i;
      if (ids.count(d->steps[3 * i + 2])) throw Error(TNB_ERR_SHAPE, "step output id reused");
      ids[d->steps[3 * i + 2]] = out;
    }
    fuse_role_pre.assign(nt, 0);
    fuse_consumer_pre.assign(nt, -1);
    auto fusable_producer = [&](int s) {
      const Pre& q = pre[s];
      if (q.smallk) return true;
      if (!q.tc) return false;
      const int64_t M = (int64_t)1 << q.rows.size(), N = (int64_t)1 << q.cols.size();
      return tc_splits(M, 2 * N, 2 * ((int64_t)1 << q.shared.size()), P->num_sms) == 1;
    };
    auto has = [](const std::vector<int64_t>& v, int64_t x) { return std::find(v.begin(), v.end(), x) != v.end(); };
    // `priority` first (in order, where present), then the rest in current order
    auto reorder = [&](std::vector<int64_t>& list, const std::vector<int64_t>& priority) {
      std::vector<int64_t> out;
      for (int64_t x : priority) if (has(list, x) && !has(out, x)) out.push_back(x);
      for (int64_t x : list) if (!has(out, x)) out.push_back(x);
      list.swap(out);
    };
    const bool fuse = fuse_env && !(d->flags & TNB_FLAG_NO_FUSE);
    struct Commit {  // copy the per-step role decisions out of the pre-pass
      std::vector<Pre>& pre;
      std::vector<char>& out;
      ~Commit() { for (size_t i = 0; i < pre.size(); ++i) out[i] = pre[i].rows_is_a ? 1 : 0; }
    } commit{pre, pre_rows_is_a};
    for (int c = d->n_steps - 1; fuse && c >= 0; --c) {
      const Pre& q = pre[c];
      if (!q.tc) continue;
      const int rows_t = q.rows_is_a ? q.a : q.b, cols_t = q.rows_is_a ? q.b : q.a;
      const int ops[2] = {rows_t, cols_t};
      int primary = -1;
      for (int r = 0; r < 2; ++r) {
        const int t = ops[r];
        if (def[t] < 0 || !fusable_producer(def[t])) continue;
        // fused-store destination indices are 32-bit half2 offsets (the
        // expanded cols operand has one more bit than the tensor)
        if ((int)sets[t].size() + (r == 1 ? 1 : 0) > 32) continue;
        fuse_role_pre[t] = r + 1;
        fuse_consumer_pre[t] = c;
        if (primary < 0) primary = t;
      }
      if (primary < 0) continue;
      // a small-K producer computes C[m][n] over gathered layouts, so its
      // m/n roles are free: put the side holding more of this consumer's
      // contracted indices on the columns (its thread-/warp-local bits)
      for (int t : ops) {
        const int p = def[t] >= 0 ? def[t] : -1;
        if (p < 0 || !fuse_role_pre[t] || !pre[p].smallk || pre[p].tc) continue;
        auto cnt = [&](const std::vector<int64_t>& side) {
          int n = 0;
          for (int64_t x : side) n += has(q.shared, x) ? 1 : 0;
          return n;
        };
        Pre& pq = pre[p];
        if (cnt(pq.rows) > cnt(pq.cols) &&
            simt_uses_smallk((int64_t)1 << pq.cols.size(), (int64_t)1 << pq.rows.size(),
                             (int64_t)1 << pq.shared.size())) {
          std::swap(pq.rows, pq.cols);
          std::swap(ord_rows[p], ord_cols[p]);
          pq.rows_is_a = false;  // SIMT: rows = b's free indices
        }
      }
      // low K bits: k0,k1 on the primary producer's result columns (n bits
      // 0,1 -> 16-B vectors), k2,k3 on its rows (lane bits: no exchange
      // needed to put destination bits 2,3 on the lanes); fall back to the
      // other side when one side has too few contracted indices
      // (a small-K SIMT producer's thread-/warp-local bits are all columns:
      // 4 per thread, 128 per warp, so every low K bit goes there first)
      const Pre& pp = pre[def[primary]];
      std::vector<int64_t> kc, kr, kpri;
      // joint choice when the other operand comes from a large small-K
      // producer: k0,k1 on both producers' columns, k2,k3 on the small-K
      // producer's columns (its fused stores need all four there)
      const int sec = (primary == rows_t && fuse_role_pre[cols_t]) ? cols_t : -1;
      if (sec >= 0 && pre[def[sec]].smallk && !pre[def[sec]].tc &&
          pre[def[sec]].rows.size() + pre[def[sec]].cols.size() > 20) {
        const Pre& ps = pre[def[sec]];
        std::vector<int64_t> both, sonly;
        for (int64_t x : ord_k[c])
          if (has(ps.cols, x)) (has(pp.cols, x) ? both : sonly).push_back(x);
        if (both.size() >= 2 && both.size() + sonly.size() >= (size_t)kKBlockLog) {
          kpri = {both[0], both[1]};
          for (int64_t x : sonly) if (kpri.size() < (size_t)kKBlockLog) kpri.push_back(x);
          for (size_t x = 2; x < both.size() && kpri.size() < (size_t)kKBlockLog; ++x) kpri.push_back(both[x]);
        }
      }
      if (kpri.empty()) {
        for (int64_t x : ord_k[c]) (has(pp.cols, x) ? kc : kr).push_back(x);
        size_t ic = 0, ir = 0;
        for (int slot = 0; slot < 4 && (ic < kc.size() || ir < kr.size()); ++slot) {
          const bool want_col = slot < 2 || pp.smallk;
          if ((want_col && ic < kc.size()) || ir >= kr.size()) kpri.push_back(kc[ic++]);
          else kpri.push_back(kr[ir++]);
        }
      }
      reorder(ord_k[c], kpri);
      const size_t L = std::min<size_t>(ord_k[c].size(), (size_t)kKBlockLog);
      for (int r = 0; r < 2; ++r) {
        const int t = ops[r];
        if (!fuse_role_pre[t]) continue;
        // destination bits of the consumer's operand, lowest first: low K
        // bits, then the consumer's free bits on that side (its result order)
        std::vector<int64_t> pri(ord_k[c].begin(), ord_k[c].begin() + L);
        const auto& side = r == 0 ? ord_rows[c] : ord_cols[c];
        pri.insert(pri.end(), side.begin(), side.end());
        const int p = def[t];
        reorder(ord_cols[p], pri);
        reorder(ord_rows[p], pri);
        if (pre[p].smallk && !pre[p].tc) {
          // a small-K producer's warp writes 32 lanes x 4 consecutive columns:
          // fuse only if its lowest columns are the consumer's lowest
          // destination bits (k0..k3, then -- rows operand -- the first row
          // bit), so a warp store covers whole 128-B lines; small results
          // are fused regardless (their staging launch costs more)
          const auto& pc = ord_cols[p];
          const size_t need = L;  // 64-B runs per 4 lanes
          bool good = L == (size_t)kKBlockLog && pc.size() >= need + 2;
          for (size_t x = 0; good && x < need; ++x) good = pc[x] == pri[x];
          const size_t bits = pre[p].rows.size() + pre[p].cols.size();
          if (!good && bits > 20) {
            fuse_role_pre[t] = 0;
            fuse_consumer_pre[t] = -1;
          }
        }
      }
    }
  }
  return op;
}

// ---------------------------------------------------------------------------
Program* program_create(const tnb_program_desc* d) {
  if (!d) throw Error(TNB_ERR_ARG, "null descriptor");
  if (d->precision != TNB_SINGLE && d->precision != TNB_DOUBLE)
    throw Error(TNB_ERR_ARG, "precision must be TNB_SINGLE or TNB_DOUBLE");
  if (d->n_leaves <= 0) throw Error(TNB_ERR_SHAPE, "program needs at least one leaf");
  if (d->n_sliced < 0 || d->n_sliced > 64) throw Error(TNB_ERR_ARG, "n_sliced must be in [0, 64]");
  int ndev = 0;
  TNB_CUDA(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) throw Error(TNB_ERR_NODEV, "device ordinal out of range");

  std::unique_ptr<Program> P(new Program());
  P->device = d->device;
  P->precision = d->precision;
  P->flags = d->flags;
  P->esize = d->precision == TNB_SINGLE ? 8 : 16;
  P->n_sliced = d->n_sliced;
  P->reuse = (d->flags & TNB_FLAG_REUSE_SLICES) != 0;
  TNB_CUDA(cudaSetDevice(P->device));
  TNB_CUDA(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device));
  TNB_CUDA(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
  const bool use_tc = d->precision == TNB_SINGLE && !(d->flags & TNB_FLAG_NO_TENSOR_CORES) &&
                      tc_available(P->device);

  // sliced index -> mask bit (engine.py:276-279: bit n_e-1-pos pins sliced[pos])
  std::unordered_map<int64_t, int> slice_bit;
  for (int i = 0; i < d->n_sliced; ++i) {
    if (slice_bit.count(d->sliced[i])) throw Error(TNB_ERR_ARG, "duplicate sliced index");
    slice_bit[d->sliced[i]] = d->n_sliced - 1 - i;
  }

  // ---- leaves
  std::unordered_map<int64_t, int> id2t;
  std::vector<SlicedLeafDesc> sl_descs;
  std::vector<uint32_t> keep;
  int64_t leaf_off = 0, slice_off = 0, idx_off = 0;
  P->leaf_ranks.assign(d->leaf_ranks, d->leaf_ranks + d->n_leaves);
  for (int i = 0; i < d->n_leaves; ++i) {
    const int r = d->leaf_ranks[i];
    if (r < 0 || r > 32) throw Error(TNB_ERR_SHAPE, "leaf rank out of range");
    TensorRec t;
    t.leaf_pos = i;
    std::vector<int64_t> full(d->leaf_indices + idx_off, d->leaf_indices + idx_off + r);
    idx_off += r;
    std::vector<std::pair<int, uint32_t>> sl;  // (mask bit, stride)
    std::vector<int> keep_src;
    for (int ax = 0; ax < r; ++ax) {
      auto it = slice_bit.find(full[ax]);
      if (it != slice_bit.end()) {
        sl.push_back({it->second, 1u << (r - 1 - ax)});
        t.dep |= 1ull << it->second;
      } else {
        t.axes.push_back(full[ax]);
        keep_src.push_back(r - 1 - ax);
      }
    }
    P->leaf_pool_off.push_back(leaf_off);
    leaf_off += (int64_t)1 << r;
    t.elems = (int64_t)1 << t.axes.size();
    if (!sl.empty()) {
      if (sl.size() > 8) throw Error(TNB_ERR_SHAPE, "more than 8 sliced axes on one leaf");
      t.variant = true;
      t.pool = POOL_SLICE;
      t.off = slice_off;
      slice_off += align_up(t.elems, 128);
      SlicedLeafDesc sd{};
      sd.src_off = P->leaf_pool_off.back();
      sd.dst_off = t.off;
      sd.out_elems = (uint32_t)t.elems;
      sd.n_sl = (uint32_t)sl.size();
      sd.keep_lut_off = (uint32_t)keep.size();
      for (size_t j = 0; j < sl.size(); ++j) { sd.sl_bit[j] = sl[j].first; sd.sl_stride[j] = sl[j].second; }
      // out index bit p (LSB first) <-> kept axis keep_src.size()-1-p
      const int nk = (int)keep_src.size();
      for (int64_t jj = 0; jj < t.elems; ++jj) {
        uint32_t o = 0;
        for (int p = 0; p < nk; ++p)
          if ((jj >> p) & 1) o |= 1u << keep_src[nk - 1 - p];
        keep.push_back(o);
      }
      sl_descs.push_back(sd);
    } else {
      t.pool = POOL_LEAF;
      t.off = P->leaf_pool_off.back();
    }
    if (id2t.count(d->leaf_ids[i])) throw Error(TNB_ERR_SHAPE, "duplicate leaf id");
    id2t[d->leaf_ids[i]] = (int)P->tensors.size();
    P->tensors.push_back(t);
  }
  P->leaf_pool_elems = leaf_off;
  P->slice_pool_elems = slice_off;

  // ---- index orders and fused-staging edges (plan_orders)
  // tensor-core eligibility: big enough to fill 128x256 tiles and amortise
  // staging.  TNB_TC_MIN_RANK (read per program; tests lower it so small
  // random networks exercise the tensor-core and fused-staging paths)
  const int tc_min_rank = env_int("TNB_TC_MIN_RANK", 26);
  const int tc_min_k = env_int("TNB_TC_MIN_K", 3);  // log2 of the smallest shared dimension
  auto tc_eligible = [&](int na, int nb, int nab) {
    return use_tc && nab >= tc_min_k && na + nb + nab >= tc_min_rank && std::max(na, nb) >= 7 &&
           std::min(na, nb) >= 3;
  };
  OrderPlan op = plan_orders(d, P.get(), use_tc, tc_eligible);
  auto& ord_k = op.ord_k;
  auto& ord_rows = op.ord_rows;
  auto& ord_cols = op.ord_cols;
  auto& pre_rows_is_a = op.rows_is_a;
  auto& fuse_role_pre = op.fuse_role;
  auto& fuse_consumer_pre = op.fuse_consumer;


  // ---- steps: axis bookkeeping (engine.py:125-134)
  for (int i = 0; i < d->n_steps; ++i) {
    const int64_t lhs = d->steps[3 * i], rhs = d->steps[3 * i + 1], outid = d->steps[3 * i + 2];
    auto ia = id2t.find(lhs), ib = id2t.find(rhs);
    if (ia == id2t.end() || ib == id2t.end() || lhs == rhs)
      throw Error(TNB_ERR_SHAPE, "step " + std::to_string(i) + " references a missing operand");
    StepRec s;
    s.a = ia->second;
    s.b = ib->second;
    id2t.erase(ia);
    id2t.erase(id2t.find(rhs));
    const TensorRec& A = P->tensors[s.a];
    const TensorRec& B = P->tensors[s.b];
    std::vector<int64_t> shared, afree, bfree;
    for (int64_t x : A.axes)
      (std::find(B.axes.begin(), B.axes.end(), x) != B.axes.end() ? shared : afree).push_back(x);
    for (int64_t x : B.axes)
      if (std::find(A.axes.begin(), A.axes.end(), x) == A.axes.end()) bfree.push_back(x);
    const int na = (int)afree.size(), nb = (int)bfree.size(), nab = (int)shared.size();
    s.mults = std::ldexp(1.0, na + nb + nab);
    TensorRec o;
    o.variant = A.variant || B.variant;
    o.dep = A.dep | B.dep;
    if (P->reuse) {
      // an operand whose mask dependence is narrower than its consumer's can be
      // reused across consecutive masks: it needs a buffer of its own
      if (A.variant && A.dep != o.dep && A.leaf_pos < 0) P->tensors[s.a].cached = true;
      if (B.variant && B.dep != o.dep && B.leaf_pos < 0) P->tensors[s.b].cached = true;
    }
    o.def_step = i;
    s.M = (int64_t)1 << na;
    s.N = (int64_t)1 << nb;
    s.K = (int64_t)1 << nab;
    const bool tc = tc_eligible(na, nb, nab);
    if (tc) {
      // expand the smaller operand (B' doubles its size); rows = the other one
      const bool rows_is_a = ((int64_t)1 << (na + nab)) >= ((int64_t)1 << (nb + nab));
      s.kind = KIND_TC;
      // canonical orders planned by the pre-pass (lists are lowest-first;
      // the canonical bit 0 is the LAST axis of these lists)
      auto as_axes = [&](const std::vector<int64_t>& low_first, const std::vector<int64_t>& cur) {
        if (low_first.size() != cur.size()) throw Error(TNB_ERR_SHAPE, "order planning mismatch");
        return std::vector<int64_t>(low_first.rbegin(), low_first.rend());
      };
      shared = as_axes(ord_k[i], shared);
      (rows_is_a ? afree : bfree) = as_axes(ord_rows[i], rows_is_a ? afree : bfree);
      (rows_is_a ? bfree : afree) = as_axes(ord_cols[i], rows_is_a ? bfree : afree);
      s.fuse_rows = fuse_role_pre[rows_is_a ? s.a : s.b] != 0;
      s.fuse_cols = fuse_role_pre[rows_is_a ? s.b : s.a] != 0;
      if (rows_is_a) {
        s.rows_t = s.a; s.cols_t = s.b;
        o.axes = afree; o.axes.insert(o.axes.end(), bfree.begin(), bfree.end());
        s.M = (int64_t)1 << na; s.N = (int64_t)1 << nb;
        s.canon_rows = canon_bits(A.axes, afree, shared);
        s.canon_cols = canon_bits(B.axes, bfree, shared);
      } else {
        s.rows_t = s.b; s.cols_t = s.a;
        o.axes = bfree; o.axes.insert(o.axes.end(), afree.begin(), afree.end());
        s.M = (int64_t)1 << nb; s.N = (int64_t)1 << na;
        s.canon_rows = canon_bits(B.axes, bfree, shared);
        s.canon_cols = canon_bits(A.axes, afree, shared);
      }
    } else {
      s.kind = KIND_SIMT;
      if (fuse_role_pre[(int)P->tensors.size()]) {
        // fused small-K producer: planned free orders; rows = a's free
        // indices unless the pre-pass swapped the kernel's m/n roles
        const bool swapped = !pre_rows_is_a[i];
        auto& mfree = swapped ? bfree : afree;
        auto& nfree = swapped ? afree : bfree;
        if (ord_rows[i].size() != mfree.size() || ord_cols[i].size() != nfree.size())
          throw Error(TNB_ERR_SHAPE, "order planning mismatch");
        mfree.assign(ord_rows[i].rbegin(), ord_rows[i].rend());
        nfree.assign(ord_cols[i].rbegin(), ord_cols[i].rend());
        if (swapped) {  // C[m over b][n over a] = B A
          std::swap(s.a, s.b);
          std::swap(afree, bfree);
          s.M = (int64_t)1 << afree.size();
          s.N = (int64_t)1 << bfree.size();
        }
      }
      const TensorRec& SA = P->tensors[s.a];
      const TensorRec& SB = P->tensors[s.b];
      o.axes = afree; o.axes.insert(o.axes.end(), bfree.begin(), bfree.end());
      const std::vector<int> src_a = canon_bits(SA.axes, afree, shared);
      const std::vector<int> src_b = canon_bits(SB.axes, bfree, shared);
      s.lut_a = add_lut(P.get(), src_a);
      s.lut_b = add_lut(P.get(), src_b);
      static const int enum_env = env_int("TNB_SMALLK_ENUM", 3);  // 1 out-lanes, 2 src-lanes, 3 auto
      if (enum_env && simt_uses_smallk((int64_t)1 << afree.size(), (int64_t)1 << bfree.size(),
                                       (int64_t)1 << shared.size()))
        s.lut_e = add_lut(P.get(), smallk_enumeration(src_a, src_b, (int)afree.size(),
                                                      (int)bfree.size(), (int)shared.size(), enum_env));
    }
    if (o.axes.size() > 32) throw Error(TNB_ERR_SHAPE, "intermediate rank above 32");
    o.elems = (int64_t)1 << o.axes.size();
    P->tensors[s.a].last_use = i;
    P->tensors[s.b].last_use = i;
    s.out = (int)P->tensors.size();
    o.fuse_role = fuse_role_pre[s.out];
    s.fuse_consumer = fuse_consumer_pre[s.out];
    s.hoisted = !o.variant && !(d->flags & TNB_FLAG_NO_HOIST);
    P->tensors.push_back(o);
    if (id2t.count(outid)) throw Error(TNB_ERR_SHAPE, "step output id reused");
    id2t[outid] = s.out;
    P->flops_per_slice += 8.0 * s.mults;
    if (s.kind == KIND_TC) { P->tc_flops_per_slice += 8.0 * s.mults; P->n_tc++; } else P->n_simt++;
    if (s.hoisted) P->n_hoisted++;
    P->steps.push_back(s);
  }
  if (id2t.size() != 1)
    throw Error(TNB_ERR_SHAPE, std::to_string(id2t.size()) + " results left after contraction");
  P->root = id2t.begin()->second;
  const int n_steps = (int)P->steps.size();
  P->tensors[P->root].last_use = n_steps;

  // ---- root output order
  {
    const TensorRec& R = P->tensors[P->root];
    std::vector<int64_t> want(d->out_order, d->out_order + d->n_out);
    std::vector<int64_t> s1 = want, s2 = R.axes;
    std::sort(s1.begin(), s1.end());
    std::sort(s2.begin(), s2.end());
    if (s1 != s2) throw Error(TNB_ERR_SHAPE, "root indices differ from the requested output order");
    P->out_elems = R.elems;
    P->root_identity = (want == R.axes);
    P->root_lut = add_lut(P.get(), canon_bits(R.axes, want, {}));
  }

  // ---- SIMT batching, memory planning
  plan_simt_batches(P.get());
  plan_memory(P.get());

  // ---- device allocations
  auto dmalloc = [](void** p, int64_t bytes) {
    if (bytes <= 0) bytes = 256;
    TNB_CUDA(cudaMalloc(p, (size_t)bytes));
  };
  dmalloc(&P->d_leaf_pool, P->leaf_pool_elems * (int64_t)P->esize);
  dmalloc(&P->d_slice_pool, P->slice_pool_elems * (int64_t)P->esize);
  dmalloc(&P->d_persist, P->persist_elems * (int64_t)P->esize);
  dmalloc(&P->d_arena, P->arena_bytes);
  dmalloc((void**)&P->d_luts, (int64_t)P->luts.size() * sizeof(ByteLut));
  TNB_CUDA(cudaMemcpy(P->d_luts, P->luts.data(), P->luts.size() * sizeof(ByteLut), cudaMemcpyHostToDevice));
  P->n_sl_descs = (int)sl_descs.size();
  dmalloc((void**)&P->d_sl_descs, (int64_t)sl_descs.size() * sizeof(SlicedLeafDesc));
  if (!sl_descs.empty())
    TNB_CUDA(cudaMemcpy(P->d_sl_descs, sl_descs.data(), sl_descs.size() * sizeof(SlicedLeafDesc),
                        cudaMemcpyHostToDevice));
  dmalloc((void**)&P->d_keep, (int64_t)keep.size() * 4);
  if (!keep.empty())
    TNB_CUDA(cudaMemcpy(P->d_keep, keep.data(), keep.size() * 4, cudaMemcpyHostToDevice));
  // per-tensor max slots: leaves | invariant step results | variant step results
  {
    const int nt = (int)P->tensors.size();
    P->slot.assign(nt, -1);
    int next = 0;
    for (int t = 0; t < nt; ++t) if (P->tensors[t].def_step < 0) P->slot[t] = next++;
    P->inv_slot_begin = next;
    for (int t = 0; t < nt; ++t)
      if (P->tensors[t].def_step >= 0 && P->tensors[t].pool == POOL_PERSIST) P->slot[t] = next++;
    P->inv_slot_count = next - P->inv_slot_begin;
    P->var_slot_begin = next;
    for (int t = 0; t < nt; ++t) if (P->slot[t] < 0) P->slot[t] = next++;
    P->var_slot_count = next - P->var_slot_begin;
    dmalloc((void**)&P->d_tmax, (int64_t)next * 4);
    TNB_CUDA(cudaMemset(P->d_tmax, 0, (size_t)next * 4));
    // guard words share the slot numbering; the last word counts re-runs
    dmalloc((void**)&P->d_guard, (int64_t)(next + 1) * 4);
    TNB_CUDA(cudaMemset(P->d_guard, 0, (size_t)(next + 1) * 4));
  }
  // tensor-core staging tables (tiled permute + split), one per TC operand
  {
    std::vector<StageHost> hosts;
    for (auto& s : P->steps) {
      if (s.kind != KIND_TC) continue;
      if (!s.fuse_rows) {
        hosts.emplace_back();
        build_stage_tables(s.canon_rows, s.K, &hosts.back());
        s.st_rows = (int)hosts.size() - 1;
      }
      if (!s.fuse_cols) {
        hosts.emplace_back();
        build_stage_tables(s.canon_cols, s.K, &hosts.back());
        s.st_cols = (int)hosts.size() - 1;
      }
    }
    size_t n32 = 0;
    for (auto& h : hosts) n32 += 3 * h.rd_t.size();
    dmalloc((void**)&P->d_stage_u32, (int64_t)n32 * 4);
    dmalloc((void**)&P->d_stage_luts, (int64_t)hosts.size() * 2 * sizeof(ByteLut));
    std::vector<uint32_t> u32;
    u32.reserve(n32);
    std::vector<ByteLut> luts;
    for (size_t i = 0; i < hosts.size(); ++i) {
      const StageHost& h = hosts[i];
      StageTables tb;
      tb.nU = h.nU;
      tb.n_tiles = h.n_tiles;
      tb.rd_t = P->d_stage_u32 + u32.size();
      u32.insert(u32.end(), h.rd_t.begin(), h.rd_t.end());
      tb.rd_src = P->d_stage_u32 + u32.size();
      u32.insert(u32.end(), h.rd_src.begin(), h.rd_src.end());
      tb.t_dst = P->d_stage_u32 + u32.size();
      u32.insert(u32.end(), h.t_dst.begin(), h.t_dst.end());
      tb.tile_src = P->d_stage_luts + luts.size();
      luts.push_back(h.tile_src);
      tb.tile_dst = P->d_stage_luts + luts.size();
      luts.push_back(h.tile_dst);
      P->stages.push_back(tb);
    }
    if (!u32.empty())
      TNB_CUDA(cudaMemcpy(P->d_stage_u32, u32.data(), u32.size() * 4, cudaMemcpyHostToDevice));
    if (!luts.empty())
      TNB_CUDA(cudaMemcpy(P->d_stage_luts, luts.data(), luts.size() * sizeof(ByteLut), cudaMemcpyHostToDevice));
  }
  P->n_acc_slots = P->n_sliced + 3;  // counter levels + total + permuted output
  dmalloc(&P->d_acc, (int64_t)P->n_acc_slots * align_up(P->out_elems, 128) * (int64_t)P->esize);

  // ---- SIMT batch descriptors (fixed addresses)
  if (!P->batches.empty()) {
    std::vector<SimtStepDesc> descs;
    for (auto& b : P->batches) {
      int64_t blocks = 0;
      const size_t first = descs.size();
      for (int i = b.first_step; i <= b.last_step; ++i) {
        const StepRec& s = P->steps[i];
        if (s.batch != (int)(&b - P->batches.data())) continue;
        SimtStepDesc d{};
        d.A = P->tensor_ptr(s.a);
        d.B = P->tensor_ptr(s.b);
        d.C = P->tensor_ptr(s.out);
        d.M = s.M; d.N = s.N; d.K = s.K;
        d.lut_a = P->d_luts + s.lut_a;
        d.lut_b = P->d_luts + s.lut_b;
        d.max_out = P->precision == TNB_SINGLE ? P->d_tmax + P->slot[s.out] : nullptr;
        d.block0 = blocks;
        blocks += simt_tiles(s.M, s.N);
        descs.push_back(d);
      }
      b.blocks = blocks;
      b.d_descs = reinterpret_cast<SimtStepDesc*>(first);  // offset, rebased below
    }
    dmalloc((void**)&P->d_simt_descs, (int64_t)descs.size() * sizeof(SimtStepDesc));
    TNB_CUDA(cudaMemcpy(P->d_simt_descs, descs.data(), descs.size() * sizeof(SimtStepDesc),
                        cudaMemcpyHostToDevice));
    for (auto& b : P->batches) b.d_descs = P->d_simt_descs + reinterpret_cast<size_t>(b.d_descs);
  }

  // ---- tensor-core plans, fused-staging maps
  plan_tensor_core_steps(P.get());

  // ---- upload leaf values
  {
    std::vector<char> host((size_t)P->leaf_pool_elems * P->esize);
    if (P->precision == TNB_SINGLE) {
      float* h = (float*)host.data();
      for (int64_t i = 0; i < 2 * P->leaf_pool_elems; ++i) h[i] = (float)d->leaf_data[i];
    } else {
      std::memcpy(host.data(), d->leaf_data, host.size());
    }
    TNB_CUDA(cudaMemcpy(P->d_leaf_pool, host.data(), host.size(), cudaMemcpyHostToDevice));
    for (int i = 0; i < d->n_leaves; ++i) upload_leaf_max(P.get(), i, d->leaf_data + 2 * P->leaf_pool_off[i]);
  }
  return P.release();
}

void program_destroy(Program* P) { delete P; }

// max|re|,|im| of a leaf (its fp32 values): the fp16 scale bound of the leaf
// and of every sliced sub-tensor prepared from it.
void upload_leaf_max(Program* P, int leaf_pos, const double* data) {
  const int64_t n = (int64_t)1 << P->leaf_ranks[leaf_pos];
  float m = 0.f;
  for (int64_t i = 0; i < 2 * n; ++i) m = std::max(m, std::fabs((float)data[i]));
  unsigned int bits;
  std::memcpy(&bits, &m, 4);
  TNB_CUDA(cudaMemcpy(P->d_tmax + P->slot[leaf_pos], &bits, 4, cudaMemcpyHostToDevice));
}

void program_info(const Program* P, tnb_program_info* info) {
  info->out_elems = P->out_elems;
  info->flops_per_slice = P->flops_per_slice;
  info->tc_flops_per_slice = P->tc_flops_per_slice;
  info->arena_bytes = P->arena_bytes;
  info->persistent_bytes = (P->leaf_pool_elems + P->slice_pool_elems + P->persist_elems) * (int64_t)P->esize;
  info->scratch_bytes = P->scratch_bytes;
  info->n_steps_tc = P->n_tc;
  info->n_steps_simt = P->n_simt;
  info->n_steps_hoisted = P->n_hoisted;
  int k = P->n_sl_descs ? 1 : 0;
  for (size_t i = 0; i < P->steps.size(); ++i) {
    const StepRec& s = P->steps[i];
    if (s.hoisted) continue;
    if (s.kind != KIND_TC && s.batch >= 0 && (int)i != P->batches[s.batch].first_step) continue;
    k += s.kind == KIND_TC ? (1 + !s.fuse_rows + !s.fuse_cols + (s.tc.splits > 1 ? 1 : 0)) : 1;
  }
  info->kernels_per_slice = k + 1;
  info->reuse_bytes = P->reuse_bytes;
  info->n_steps_fused = 0;
  info->n_steps_fused_fast = 0;
  for (auto& s : P->steps) {
    const FuseOut& f = s.kind == KIND_TC ? s.tc.fuse : s.simt_fuse;
    if (f.mode == 0) continue;
    info->n_steps_fused++;
    info->n_steps_fused_fast += (f.fast || f.vec) ? 1 : 0;
  }
}

void program_set_leaf(Program* P, int leaf_pos, const double* data) {
  if (leaf_pos < 0 || leaf_pos >= (int)P->leaf_ranks.size()) throw Error(TNB_ERR_ARG, "leaf index out of range");
  TNB_CUDA(cudaSetDevice(P->device));
  const int64_t n = (int64_t)1 << P->leaf_ranks[leaf_pos];
  char* dst = (char*)P->d_leaf_pool + (size_t)P->leaf_pool_off[leaf_pos] * P->esize;
  if (P->precision == TNB_SINGLE) {
    std::vector<float> h(2 * n);
    for (int64_t i = 0; i < 2 * n; ++i) h[i] = (float)data[i];
    TNB_CUDA(cudaMemcpyAsync(dst, h.data(), h.size() * 4, cudaMemcpyHostToDevice, P->stream));
    TNB_CUDA(cudaStreamSynchronize(P->stream));
  } else {
    TNB_CUDA(cudaMemcpyAsync(dst, data, (size_t)n * 16, cudaMemcpyHostToDevice, P->stream));
    TNB_CUDA(cudaStreamSynchronize(P->stream));
  }
  upload_leaf_max(P, leaf_pos, data);
  P->invariant_valid = false;
}

// Batched repin: one staged host buffer, contiguous runs of leaves coalesced
// into single copies, leaf max slots uploaded in one copy, one sync.
void program_set_leaves(Program* P, int n, const int32_t* pos, const double* data) {
  const int nl = (int)P->leaf_ranks.size();
  TNB_CUDA(cudaSetDevice(P->device));
  std::vector<char> host;
  struct Run { int64_t dst_elem, n_elem; size_t host_off; };
  std::vector<Run> runs;
  std::vector<unsigned int> maxbits(nl, 0);
  int lo = nl, hi = -1;
  const double* src = data;
  for (int i = 0; i < n; ++i) {
    const int p = pos[i];
    if (p < 0 || p >= nl) throw Error(TNB_ERR_ARG, "leaf index out of range");
    const int64_t ne = (int64_t)1 << P->leaf_ranks[p];
    const size_t off = host.size();
    host.resize(off + (size_t)ne * P->esize);
    float m = 0.f;
    if (P->precision == TNB_SINGLE) {
      float* h = reinterpret_cast<float*>(host.data() + off);
      for (int64_t j = 0; j < 2 * ne; ++j) {
        h[j] = (float)src[j];
        m = std::max(m, std::fabs(h[j]));
      }
    } else {
      std::memcpy(host.data() + off, src, (size_t)ne * 16);
    }
    std::memcpy(&maxbits[p], &m, 4);
    lo = std::min(lo, p);
    hi = std::max(hi, p);
    const int64_t dst = P->leaf_pool_off[p];
    if (!runs.empty() && runs.back().dst_elem + runs.back().n_elem == dst &&
        runs.back().host_off + (size_t)runs.back().n_elem * P->esize == off)
      runs.back().n_elem += ne;
    else
      runs.push_back({dst, ne, off});
    src += 2 * ne;
  }
  for (const Run& r : runs)
    TNB_CUDA(cudaMemcpyAsync((char*)P->d_leaf_pool + (size_t)r.dst_elem * P->esize,
                             host.data() + r.host_off, (size_t)r.n_elem * P->esize,
                             cudaMemcpyHostToDevice, P->stream));
  if (hi >= lo && P->precision == TNB_SINGLE) {
    // unchanged leaves in [lo, hi] keep their slot: merge with the current values
    std::vector<unsigned int> cur(hi - lo + 1);
    TNB_CUDA(cudaMemcpyAsync(cur.data(), P->d_tmax + lo, cur.size() * 4, cudaMemcpyDeviceToHost,
                             P->stream));
    TNB_CUDA(cudaStreamSynchronize(P->stream));
    std::vector<char> touched(nl, 0);
    for (int i = 0; i < n; ++i) touched[pos[i]] = 1;
    for (int p = lo; p <= hi; ++p)
      if (touched[p]) cur[p - lo] = maxbits[p];
    TNB_CUDA(cudaMemcpyAsync(P->d_tmax + lo, cur.data(), cur.size() * 4, cudaMemcpyHostToDevice,
                             P->stream));
    TNB_CUDA(cudaStreamSynchronize(P->stream));
  } else {
    TNB_CUDA(cudaStreamSynchronize(P->stream));
  }
  P->invariant_valid = false;
}

void program_set_leaf_c64(Program* P, int leaf_pos, const float* data) {
  if (leaf_pos < 0 || leaf_pos >= (int)P->leaf_ranks.size()) throw Error(TNB_ERR_ARG, "leaf index out of range");
  if (P->precision != TNB_SINGLE) throw Error(TNB_ERR_ARG, "complex64 upload needs a single-precision program");
  TNB_CUDA(cudaSetDevice(P->device));
  const int64_t n = (int64_t)1 << P->leaf_ranks[leaf_pos];
  char* dst = (char*)P->d_leaf_pool + (size_t)P->leaf_pool_off[leaf_pos] * P->esize;
  TNB_CUDA(cudaMemcpyAsync(dst, data, (size_t)n * 8, cudaMemcpyHostToDevice, P->stream));
  launch_absmax((const float2*)dst, n, P->d_tmax + P->slot[leaf_pos], P->stream);
  TNB_CUDA(cudaStreamSynchronize(P->stream));
  P->invariant_valid = false;
}

void program_set_leaf_device(Program* P, int leaf_pos, const void* dev) {
  if (leaf_pos < 0 || leaf_pos >= (int)P->leaf_ranks.size()) throw Error(TNB_ERR_ARG, "leaf index out of range");
  TNB_CUDA(cudaSetDevice(P->device));
  const int64_t n = (int64_t)1 << P->leaf_ranks[leaf_pos];
  char* dst = (char*)P->d_leaf_pool + (size_t)P->leaf_pool_off[leaf_pos] * P->esize;
  TNB_CUDA(cudaMemcpyAsync(dst, dev, (size_t)n * P->esize, cudaMemcpyDeviceToDevice, P->stream));
  if (P->precision == TNB_SINGLE)
    launch_absmax((const float2*)dst, n, P->d_tmax + P->slot[leaf_pos], P->stream);
  TNB_CUDA(cudaStreamSynchronize(P->stream));
  P->invariant_valid = false;
}

namespace {

struct EvRec { int cls; cudaEvent_t a, b; };

struct RunCtx {
  Program* P;
  std::vector<EvRec> recs;
  size_t ev_next = 0;
  int64_t launches = 0, gemm_launches = 0, reused = 0;
  double gemm_flops = 0;
  cudaEvent_t get() {
    if (ev_next == P->ev_pool.size()) {
      cudaEvent_t e;
      TNB_CUDA(cudaEventCreate(&e));
      P->ev_pool.push_back(e);
    }
    return P->ev_pool[ev_next++];
  }
  // timing 1: every kernel class; timing 2: GEMM launches + the range total
  // only (no event records around the hundreds of tiny kernels, whose issue
  // cost would otherwise show up in the measured time)
  bool records(int cls) const { return P->timing == 1 || (P->timing == 2 && cls <= 0); }
  cudaEvent_t mark(int cls = -1) {
    if (!records(cls)) return nullptr;
    cudaEvent_t e = get();
    TNB_CUDA(cudaEventRecord(e, P->stream));
    return e;
  }
  void close(int cls, cudaEvent_t a) {
    if (!a || !records(cls)) return;
    cudaEvent_t b = mark(cls);
    recs.push_back({cls, a, b});
  }
};

thread_local RunCtx* g_ctx = nullptr;

template <typename T>
void exec_step(Program* P, StepRec& s, int parts) {
  RunCtx& C = *g_ctx;
  if (s.kind == KIND_SIMT && !(parts & kPre)) return;
  if (s.kind == KIND_SIMT && s.batch >= 0) {
    const Program::SimtBatch& b = P->batches[s.batch];
    if (&s - P->steps.data() != b.first_step) return;  // launched with its batch
    cudaEvent_t e = C.mark(2);
    launch_contract_simt_batch<T>(b.d_descs, b.n, b.blocks, P->stream);
    C.close(2, e);
    C.launches++;
    return;
  }
  if (s.kind == KIND_SIMT && s.dstage) {
    cudaEvent_t e = C.mark(2);
    T* ac = (T*)((char*)P->d_arena + s.scratch_off);
    T* bc = (T*)((char*)P->d_arena + s.scratch_off + align_up(s.M * s.K * 16, kAlign));
    const ByteLut* id = P->d_luts + P->lut_ident;
    launch_permute<T>((const T*)P->tensor_ptr(s.a), ac, s.M * s.K, P->d_luts + s.lut_a, P->stream);
    launch_permute<T>((const T*)P->tensor_ptr(s.b), bc, s.N * s.K, P->d_luts + s.lut_b, P->stream);
    launch_contract_simt<T>(ac, bc, (T*)P->tensor_ptr(s.out), s.M, s.N, s.K, id, id, nullptr,
                            nullptr, nullptr, P->stream);
    C.close(2, e);
    C.launches += 3;
    return;
  }
  if (s.kind == KIND_SIMT) {
    cudaEvent_t e = C.mark(2);
    launch_contract_simt<T>((const T*)P->tensor_ptr(s.a), (const T*)P->tensor_ptr(s.b),
                            (T*)P->tensor_ptr(s.out), s.M, s.N, s.K, P->d_luts + s.lut_a,
                            P->d_luts + s.lut_b, s.lut_e >= 0 ? P->d_luts + s.lut_e : nullptr,
                            P->precision == TNB_SINGLE ? P->d_tmax + P->slot[s.out] : nullptr,
                            s.simt_fuse.mode ? &s.simt_fuse : nullptr, P->stream);
    C.launches++;
    if (s.has_redo) {
      launch_contract_simt<T>((const T*)P->tensor_ptr(s.a), (const T*)P->tensor_ptr(s.b),
                              (T*)P->tensor_ptr(s.out), s.M, s.N, s.K, P->d_luts + s.lut_a,
                              P->d_luts + s.lut_b, s.lut_e >= 0 ? P->d_luts + s.lut_e : nullptr,
                              P->d_tmax + P->slot[s.out], &s.simt_redo, P->stream);
      C.launches += 1;
    }
    C.close(2, e);
    return;
  }
  if constexpr (std::is_same<T, float2>::value) {
    const int64_t Kp = 2 * s.K, Np = 2 * s.N;
    const float2* rows = (const float2*)P->tensor_ptr(s.rows_t);
    const float2* cols = (const float2*)P->tensor_ptr(s.cols_t);
    // staging destinations: the step's scratch, rows planes first (same
    // layout as the plan's TMA maps; fused operands are not staged here)
    char* base = (char*)P->d_arena + s.scratch_off;
    __half* ahi = (__half*)base;
    __half* alo = ahi + s.M * Kp;
    __half* bhi = (__half*)(base + (s.fuse_rows ? 0 : 2 * s.M * Kp * 2));
    __half* blo = bhi + Np * Kp;
    cudaEvent_t e = nullptr;
    if ((parts & kPre) && (!s.fuse_rows || !s.fuse_cols)) {
      e = C.mark(1);
      if (!s.fuse_rows) {
        launch_stage(rows, P->stages[s.st_rows], s.K, false, P->d_tmax + P->slot[s.rows_t], ahi, alo, P->stream);
        C.launches++;
      }
      if (!s.fuse_cols) {
        launch_stage(cols, P->stages[s.st_cols], s.K, true, P->d_tmax + P->slot[s.cols_t], bhi, blo, P->stream);
        C.launches++;
      }
      C.close(1, e);
    }
    if (parts & kGemm) {
      e = C.mark(0);
      tc_launch_gemm(&s.tc, P->stream);
      C.close(0, e);
      C.launches += 1;
      C.gemm_launches++;
      C.gemm_flops += 8.0 * s.mults;
      if (s.has_redo) {
        // scale-guard re-run (exits at once unless the guard fires)
        e = C.mark(1);
        tc_launch_gemm(&s.tc_redo, P->stream);
        C.close(1, e);
        C.launches += 1;
      }
    }
    if ((parts & kPost) && s.tc.splits > 1) {
      e = C.mark(1);
      launch_splitk_reduce(s.tc.C, s.tc.splits, s.M * Np, (float*)P->tensor_ptr(s.out),
                           s.tc.scale_rows, s.tc.scale_cols, s.tc.max_out, P->stream);
      C.close(1, e);
      C.launches++;
    }
  } else {
    throw Error(TNB_ERR_ARG, "tensor-core path requires single precision");
  }
}

// Capture the per-slice launch sequence (everything but the GEMMs) into
// graph segments: [max-slot reset, SIMT/staging kernels ...] GEMM [split-K
// reduce, SIMT/staging ...] GEMM ...  Capturing records without executing.
template <typename T>
void build_segments(Program* P) {
  RunCtx& C = *g_ctx;
  cudaStream_t st = P->stream;
  const int64_t launches0 = C.launches;
  int64_t seg_start = C.launches;
  auto begin = [&] {
    TNB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    seg_start = C.launches;
  };
  auto end = [&] {
    cudaGraph_t g = nullptr;
    TNB_CUDA(cudaStreamEndCapture(st, &g));
    size_t nodes = 0;
    TNB_CUDA(cudaGraphGetNodes(g, nullptr, &nodes));
    if (nodes > 0) {
      Program::Segment seg;
      TNB_CUDA(cudaGraphInstantiate(&seg.exec, g, 0));
      seg.kernels = (int)(C.launches - seg_start);
      P->items.push_back({(int)P->segs.size(), -1});
      P->segs.push_back(seg);
    }
    TNB_CUDA(cudaGraphDestroy(g));
  };
  P->items.clear();
  begin();
  if (P->var_slot_count)
    TNB_CUDA(cudaMemsetAsync(P->d_tmax + P->var_slot_begin, 0, (size_t)P->var_slot_count * 4, st));
  for (size_t i = 0; i < P->steps.size(); ++i) {
    StepRec& s = P->steps[i];
    if (s.hoisted) continue;
    if (s.kind != KIND_TC) {
      exec_step<T>(P, s, kPre);
      continue;
    }
    exec_step<T>(P, s, kPre);
    end();
    P->items.push_back({-1, (int)i});
    begin();
    exec_step<T>(P, s, kPost);
  }
  end();
  C.launches = launches0;  // nothing ran: the replays count their kernels
  P->segs_built = true;
}

template <typename T>
void run_range_t(Program* P, uint64_t a, uint64_t b, int mode, void* out, bool out_dev) {
  RunCtx ctx;
  ctx.P = P;
  g_ctx = &ctx;
  struct Reset { ~Reset() { g_ctx = nullptr; } } reset;
  cudaStream_t st = P->stream;
  const int64_t E = P->out_elems;
  const int64_t slot_stride = align_up(E, 128);
  T* slots = (T*)P->d_acc;
  auto slot = [&](int i) { return slots + (size_t)i * slot_stride; };
  T* total_slot = slot(P->n_sliced + 1);
  T* perm_slot = slot(P->n_sliced + 2);
  // CUDA-graph segments for the per-slice launches (not with per-class
  // timing, whose events would be baked into the graphs, nor reuse mode,
  // which skips steps per mask)
  static const int graphs_env = env_int("TNB_GRAPHS", 1);
  const bool use_graphs = graphs_env && P->timing != 1 && !P->reuse;
  cudaEvent_t t_start = ctx.mark(-1);
  unsigned int* redo_count = P->d_guard + P->slot.size();
  TNB_CUDA(cudaMemsetAsync(redo_count, 0, 4, st));

  // hoisted slice-invariant steps (once per leaf-data version)
  if (!P->invariant_valid) {
    if (P->inv_slot_count)
      TNB_CUDA(cudaMemsetAsync(P->d_tmax + P->inv_slot_begin, 0, (size_t)P->inv_slot_count * 4, st));
    for (auto& s : P->steps) {
      if (s.hoisted) exec_step<T>(P, s);
      s.has_key = false;  // leaf data changed: every cached result is stale
    }
    P->invariant_valid = true;
  }

  // occupied binary-counter levels; level l holds a sum of 2^l chunks
  std::vector<int> occupied(P->n_sliced + 2, 0);
  uint64_t count = 0;
  const T* root_ptr = (const T*)P->tensor_ptr(P->root);
  for (uint64_t mask = a; mask < b; ++mask) {
    cudaEvent_t e = ctx.mark(3);
    launch_prepare_leaves<T>((const T*)P->d_leaf_pool, (T*)P->d_slice_pool, P->d_sl_descs,
                             P->n_sl_descs, P->d_keep, mask, st);
    if (P->n_sl_descs) ctx.launches++;
    ctx.close(3, e);
    if (!P->reuse && use_graphs) {
      if (!P->segs_built) build_segments<T>(P);
      for (const auto& it : P->items) {
        if (it.seg >= 0) {
          TNB_CUDA(cudaGraphLaunch(P->segs[it.seg].exec, st));
          ctx.launches += P->segs[it.seg].kernels;
        } else {
          exec_step<T>(P, P->steps[it.step], kGemm);
        }
      }
    } else if (!P->reuse) {
      if (P->var_slot_count)
        TNB_CUDA(cudaMemsetAsync(P->d_tmax + P->var_slot_begin, 0, (size_t)P->var_slot_count * 4, st));
      for (auto& s : P->steps)
        if (!s.hoisted) exec_step<T>(P, s);
    } else {
      // cross-slice reuse: a step re-executes only when the mask bits its
      // result depends on change; skipped results are bit-identical to a
      // recomputation (deterministic kernels, fresh fp16 scale per result)
      for (auto& s : P->steps) {
        if (s.hoisted) continue;
        const uint64_t key = mask & P->tensors[s.out].dep;
        if (s.has_key && s.last_key == key) { ctx.reused++; continue; }
        TNB_CUDA(cudaMemsetAsync(P->d_tmax + P->slot[s.out], 0, 4, st));
        exec_step<T>(P, s);
        s.has_key = true;
        s.last_key = key;
      }
    }
    e = ctx.mark(3);
    if (mode == TNB_FIXED) {
      // binary-counter increment: the new chunk merges with the levels
      // 0..merges-1 (x = prev + x, lowest level first) -> level `merges`
      int merges = 0;
      while ((count >> merges) & 1ull) ++merges;
      launch_counter_merge<T>(root_ptr, slot(0), slot_stride, merges, slot(merges), E, st);
      for (int l = 0; l < merges; ++l) occupied[l] = 0;
      occupied[merges] = 1;
    } else {
      // free mode: data = x if data is None else data + x (engine.py:295-298)
      if (count == 0) launch_copy<T>(root_ptr, total_slot, E, st);
      else launch_add<T>(total_slot, root_ptr, total_slot, E, st);
    }
    ctx.launches++;
    ctx.close(3, e);
    ++count;
  }
  cudaEvent_t e = ctx.mark(3);
  const T* result = total_slot;
  if (mode == TNB_FIXED) {
    // total = stack[0] (highest level) + stack[1] + ... (engine.py:218-221)
    bool first = true;
    for (int l = (int)occupied.size() - 1; l >= 0; --l) {
      if (!occupied[l]) continue;
      if (first) launch_copy<T>(slot(l), total_slot, E, st);
      else launch_add<T>(total_slot, slot(l), total_slot, E, st);
      first = false;
      ctx.launches++;
    }
  }
  if (!P->root_identity) {
    launch_permute<T>(result, perm_slot, E, P->d_luts + P->root_lut, st);
    ctx.launches++;
    result = perm_slot;
  }
  ctx.close(3, e);
  if (out_dev) {
    TNB_CUDA(cudaMemcpyAsync(out, result, (size_t)E * sizeof(T), cudaMemcpyDeviceToDevice, st));
  } else {
    TNB_CUDA(cudaMemcpyAsync(out, result, (size_t)E * sizeof(T), cudaMemcpyDeviceToHost, st));
  }
  cudaEvent_t t_end = ctx.mark(-1);
  unsigned int redos = 0;
  TNB_CUDA(cudaMemcpyAsync(&redos, redo_count, 4, cudaMemcpyDeviceToHost, st));
  TNB_CUDA(cudaStreamSynchronize(st));
  if (std::is_same<T, float2>::value && getenv("TNB_DEBUG_MAX")) {
    // diagnostic: per-step output max vs the a-priori bound 2 K max|A| max|B|
    std::vector<float> mx(P->slot.size() ? *std::max_element(P->slot.begin(), P->slot.end()) + 1 : 0);
    TNB_CUDA(cudaMemcpy(mx.data(), P->d_tmax, mx.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < P->steps.size(); ++i) {
      const StepRec& s = P->steps[i];
      const float ma = mx[P->slot[s.a]], mb = mx[P->slot[s.b]], mc = mx[P->slot[s.out]];
      const double bound = 2.0 * (double)s.K * ma * mb;
      fprintf(stderr, "TNB_MAX step %zu kind %d M %lld N %lld K %lld maxA %.3e maxB %.3e maxC %.3e log2(bound/maxC) %.2f\n",
              i, s.kind, (long long)s.M, (long long)s.N, (long long)s.K, ma, mb, mc,
              mc > 0 ? std::log2(bound / mc) : -1.0);
    }
  }
  tnb_timing tm{};
  if (P->timing) {
    float ms = 0;
    TNB_CUDA(cudaEventElapsedTime(&ms, t_start, t_end));
    tm.total_ms = ms;
    for (auto& r : ctx.recs) {
      TNB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      if (r.cls == 0) tm.gemm_ms += ms;
      else if (r.cls == 1) tm.convert_ms += ms;
      else if (r.cls == 2) tm.simt_ms += ms;
      else tm.other_ms += ms;
    }
  }
  tm.launches = ctx.launches;
  tm.gemm_launches = ctx.gemm_launches;
  tm.gemm_flops = ctx.gemm_flops;
  tm.steps_reused = ctx.reused;
  tm.scale_redos = redos;
  P->last = tm;
}

}  // namespace

void program_run_range(Program* P, uint64_t a, uint64_t b, int mode, void* out, int out_dev) {
  if (mode != TNB_FIXED && mode != TNB_FREE) throw Error(TNB_ERR_ARG, "unknown reduction mode");
  const uint64_t total = P->n_sliced >= 64 ? ~0ull : (1ull << P->n_sliced);
  if (!(a < b) || (P->n_sliced < 64 && b > total))
    throw Error(TNB_ERR_RANGE, "range [" + std::to_string(a) + "," + std::to_string(b) +
                                   ") outside [0," + std::to_string(total) + ")");
  if (!out) throw Error(TNB_ERR_ARG, "null output");
  TNB_CUDA(cudaSetDevice(P->device));
  if (P->precision == TNB_SINGLE) run_range_t<float2>(P, a, b, mode, out, out_dev != 0);
  else run_range_t<double2>(P, a, b, mode, out, out_dev != 0);
}

void program_set_timing(Program* P, int on) { P->timing = on < 0 ? 0 : (on > 2 ? 1 : on); }
void program_get_timing(const Program* P, tnb_timing* t) { *t = P->last; }

}  // namespace tnb
