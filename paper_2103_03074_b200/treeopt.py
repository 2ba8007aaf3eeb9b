"""B200-aware head-tree / slice co-optimisation.

``select_slices_b200(tn, tree, target_space, ...)`` is a drop-in for the
reference's ``select_slices`` (tncut/slicing.py:76-196): same inputs, same
``(SlicePlan, ContractionTree)`` result (the reference's own classes when
``tncut`` is importable), and the returned tree keeps the reference's
first-cut structure (head = lhs subtree of the final step,
ordering.py:99-147), the same head leaves and the same cut legs, so
``compute_head_vector`` / ``compute_tail_amplitudes`` (reference or this
executor) consume it unchanged and produce the same head vector.

What differs is the objective.  The reference slices on space alone and
rebuilds the worst subtree greedily; here the head's pairwise order and
its sliced set are searched jointly for the TOTAL head work
``2^n_e * tc(slice)`` under the space target (``csrc/treeopt.cpp``,
native, multi-threaded; C-ABI ``include/tnb_plan.h``).  With
``objective="b200"`` the step cost is the executor's time model
(tensor-core GEMM rate, HBM rate and a fixed per-step cost) instead of the
multiplication count.  The caller's tree and sliced set are always
candidates, so the result is never worse than the input under the chosen
objective.

The plan is host-side planning, not the data path; it never touches the
GPU and runs where ``tncut`` is absent.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import subprocess

import numpy as np

from .planner import step_mults

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtnbplan.so")
SRC = os.path.join(_PKG, "csrc", "treeopt.cpp")
HDR = os.path.join(os.path.dirname(_PKG), "include", "tnb_plan.h")


class Options(ctypes.Structure):  # tnb_plan.h: tnbp_options
    _fields_ = [
        ("target_log2", ctypes.c_int),
        ("trials", ctypes.c_int),
        ("keep_top", ctypes.c_int),
        ("reconf_k", ctypes.c_int),
        ("polish_k", ctypes.c_int),
        ("threads", ctypes.c_int),
        ("objective", ctypes.c_int),
        ("seed", ctypes.c_uint64),
        ("gemm_flops", ctypes.c_double),
        ("hbm_bytes", ctypes.c_double),
        ("step_s", ctypes.c_double),
        ("time_budget_s", ctypes.c_double),
        ("slice_repeats", ctypes.c_int),
        ("keep_slices", ctypes.c_int),
    ]


EXPORTS = ("tnbp_optimize", "tnbp_order", "tnbp_tree_cost", "tnbp_default_options",
           "tnbp_last_error")


def build(force: bool = False) -> str:
    """g++ build of libtnbplan.so (host code only; no GPU needed)."""
    stale = force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(p) > os.path.getmtime(LIB_PATH) for p in (SRC, HDR))
    if stale:
        tmp = LIB_PATH + ".tmp"
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", SRC, "-o", tmp]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed ({' '.join(cmd)}):\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built (python -m paper_2103_03074_b200.build)")
        lib = ctypes.CDLL(LIB_PATH)
        ip = ctypes.POINTER(ctypes.c_int)
        lib.tnbp_optimize.argtypes = [ctypes.c_int, ip, ip, ctypes.c_int, ctypes.c_char_p, ip, ip,
                                      ctypes.c_int, ctypes.POINTER(Options), ip, ip, ip,
                                      ctypes.POINTER(ctypes.c_double)]
        lib.tnbp_tree_cost.argtypes = [ctypes.c_int, ip, ip, ctypes.c_int, ip, ip, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        lib.tnbp_order.argtypes = [ctypes.c_int, ip, ip, ctypes.c_int, ctypes.POINTER(Options), ip,
                                   ctypes.POINTER(ctypes.c_double)]
        lib.tnbp_default_options.argtypes = [ctypes.POINTER(Options)]
        lib.tnbp_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


# ------------------------------------------------------------------ types

try:  # pragma: no cover - environment dependent
    from tncut.ordering import Complexity  # type: ignore
    from tncut.slicing import SlicePlan  # type: ignore
except Exception:

    @dataclasses.dataclass
    class Complexity:  # ordering.py:54-60
        tc: int
        sc_log2: int
        per_step: list

    @dataclasses.dataclass
    class SlicePlan:  # slicing.py:35-46
        sliced_indices: list
        per_subtask: Complexity
        overhead: float
        target_space: int | None = None
        tail_per_assignment: Complexity | None = None

        @property
        def subtask_count(self) -> int:
            return 1 << len(self.sliced_indices)


@dataclasses.dataclass
class HeadProblem:
    """The head network in the optimiser's dense encoding."""
    head_leaves: list        # node ids, position = dense leaf id
    index_ids: list          # dense index id -> network index id
    leaf_ptr: np.ndarray
    leaf_idx: np.ndarray
    sliceable: np.ndarray    # uint8 per dense index: both endpoints in the head
    init_children: np.ndarray  # the caller's head tree, SSA children

    @property
    def n(self) -> int:
        return len(self.head_leaves)


def head_problem(tn, tree) -> HeadProblem:
    if tree.first_cut is None:
        raise ValueError("select_slices_b200 needs a first-cut (head/tail) tree")
    head, _ = tree.head_tail_leaves()
    head_leaves = sorted(head)
    pos = {nid: i for i, nid in enumerate(head_leaves)}
    index_ids = sorted({ix for nid in head_leaves for ix in tn.nodes[nid].indices})
    dense = {ix: k for k, ix in enumerate(index_ids)}
    ptr = [0]
    idx = []
    for nid in head_leaves:
        idx.extend(dense[ix] for ix in tn.nodes[nid].indices)
        ptr.append(len(idx))
    hs = set(head_leaves)
    sliceable = np.zeros(len(index_ids), np.uint8)
    for ix, k in dense.items():
        eps = tn.index_endpoints.get(ix, ())
        if len(eps) == 2 and eps[0] in hs and eps[1] in hs:  # slicing.py:97-102
            sliceable[k] = 1
    ssa = dict(pos)
    ch = []
    for i, s in enumerate(tree.head_steps()):
        ch += [ssa[s.lhs], ssa[s.rhs]]
        ssa[s.out] = len(head_leaves) + i
    return HeadProblem(head_leaves, index_ids, np.asarray(ptr, np.int32),
                       np.asarray(idx, np.int32), sliceable, np.asarray(ch, np.int32))


def order_network(index_sets: dict, next_out: int, *, cap_log2: int = 30,
                  objective: str = "b200", exact_k: int = 14, stats: dict | None = None) -> list:
    """Pairwise order of a whole small network {leaf id: indices} ->
    [(lhs, rhs, out)] with out ids next_out, next_out + 1, ... (``tnbp_order``).

    A deterministic size-reduction greedy, then every subtree of <= exact_k
    operands re-optimised exactly under the B200 time model (the whole order
    when the network has <= exact_k leaves), never creating a tensor above
    max(cap_log2, the greedy's largest).  Indices with one endpoint stay
    open.  Used for the head-absorbed tail, which the reference never builds
    (its blocked tail is ordered by ordering.py:256-285's greedy)."""
    ids = sorted(index_sets)
    if len(ids) < 2:
        return []
    dense: dict = {}
    ptr = [0]
    idx = []
    for nid in ids:
        for ix in index_sets[nid]:
            idx.append(dense.setdefault(ix, len(dense)))
        ptr.append(len(idx))
    lp, li = np.asarray(ptr, np.int32), np.asarray(idx or [0], np.int32)
    opt = Options()
    lib = load()
    lib.tnbp_default_options(ctypes.byref(opt))
    opt.target_log2 = int(cap_log2)
    opt.polish_k = int(exact_k)
    opt.objective = _objective(objective)
    opt.time_budget_s = 30.0
    n = len(ids)
    ch = np.zeros(2 * (n - 1), np.int32)
    st = (ctypes.c_double * 3)()
    rc = lib.tnbp_order(n, _ptr(lp), _ptr(li), len(dense), ctypes.byref(opt), _ptr(ch), st)
    if rc:
        raise ValueError(lib.tnbp_last_error().decode())
    if stats is not None:
        stats.update(log2_cost=st[0], sc=int(st[1]), log2_mults=st[2])
    names = list(ids)
    steps = []
    for i in range(n - 1):
        out = next_out + i
        steps.append((names[ch[2 * i]], names[ch[2 * i + 1]], out))
        names.append(out)
    return steps


def tree_cost(tn, tree, sliced, objective: str = "mults") -> tuple:
    """(log2 cost per slice, max rank, log2 total) of the head under the native model."""
    hp = head_problem(tn, tree)
    dense = {ix: k for k, ix in enumerate(hp.index_ids)}
    sl = np.asarray([dense[ix] for ix in sliced], np.int32)
    out = (ctypes.c_double * 3)()
    lib = load()
    rc = lib.tnbp_tree_cost(hp.n, _ptr(hp.leaf_ptr), _ptr(hp.leaf_idx), len(hp.index_ids),
                            _ptr(hp.init_children), _ptr(sl) if len(sl) else None, len(sl),
                            _objective(objective), out)
    if rc:
        raise RuntimeError(lib.tnbp_last_error().decode())
    return out[0], int(out[1]), out[2]


def _objective(name: str) -> int:
    if name in ("mults", "tc", "flops"):
        return 0
    if name == "b200":
        return 1
    raise ValueError(f"unknown objective {name!r} (mults | b200)")


def select_slices_b200(tn, tree, target_space: int, *, objective: str = "mults",
                       trials: int = 1024, keep_top: int = 16, reconf_k: int = 10,
                       polish_k: int = 12, slice_repeats: int = 2, threads: int = 0,
                       seed: int = 0, time_budget_s: float = 60.0,
                       initial_slices=None, gemm_flops: float = 4.1e14,
                       hbm_bytes: float | None = None, step_s: float = 5e-6, stats: dict | None = None,
                       restarts: int = 1, keep_slices: bool = False):
    """Drop-in for ``tncut.slicing.select_slices`` (slicing.py:76-196).

    Returns ``(SlicePlan, ContractionTree)``.  ``initial_slices`` (e.g. the
    reference's own plan for ``tree``) is kept as a candidate.  ``stats``
    receives the optimiser's figures (log2 costs, seconds, candidates).
    ``restarts`` runs the search with seeds seed, seed+1, ... and keeps the
    cheapest plan: the greedy slicing path is seed-sensitive (C4 at 2^30:
    2^69.8 - 2^77.0 total over seeds 0-6).  ``keep_slices`` (with
    ``initial_slices``) keeps the caller's sliced set and only re-optimises
    the head tree's order: the same slices (same mask -> same partial head
    vector), computed by a cheaper tree.
    """
    if restarts > 1:
        best = None
        for r in range(restarts):
            st: dict = {}
            res = select_slices_b200(tn, tree, target_space, objective=objective, trials=trials,
                                     keep_top=keep_top, reconf_k=reconf_k, polish_k=polish_k,
                                     slice_repeats=slice_repeats, threads=threads, seed=seed + r,
                                     time_budget_s=time_budget_s, initial_slices=initial_slices,
                                     gemm_flops=gemm_flops, hbm_bytes=hbm_bytes, step_s=step_s,
                                     stats=st, keep_slices=keep_slices)
            if best is None or st["log2_total"] < best[1]["log2_total"]:
                best = (res, dict(st, seed=seed + r))
        if stats is not None:
            stats.update(best[1], restarts=restarts)
        return best[0]
    if hbm_bytes is None:  # model bandwidth (bytes/s); TNB_MODEL_BW overrides
        hbm_bytes = float(os.environ.get("TNB_MODEL_BW", "4.0e12"))
    if keep_slices and not initial_slices:
        raise ValueError("keep_slices needs initial_slices (the sliced set to keep)")
    hp = head_problem(tn, tree)
    dense = {ix: k for k, ix in enumerate(hp.index_ids)}
    unknown = [ix for ix in (initial_slices or []) if ix not in dense]
    if unknown:
        from .errors import ShapeMismatch
        raise ShapeMismatch(f"sliced indices {unknown[:4]} are not head indices")
    init_sl = np.asarray([dense[ix] for ix in (initial_slices or [])], np.int32)
    opt = Options()
    lib = load()
    lib.tnbp_default_options(ctypes.byref(opt))
    opt.target_log2 = int(target_space)
    opt.trials = int(trials)
    opt.keep_top = int(keep_top)
    opt.reconf_k = int(reconf_k)
    opt.polish_k = int(polish_k)
    opt.threads = int(threads) if threads else int(os.environ.get("TNB_PLAN_THREADS", "0") or 0)
    opt.objective = _objective(objective)
    opt.seed = int(seed)
    opt.gemm_flops = float(gemm_flops)
    opt.hbm_bytes = float(hbm_bytes)
    opt.step_s = float(step_s)
    opt.time_budget_s = float(time_budget_s)
    opt.slice_repeats = int(slice_repeats)
    opt.keep_slices = int(bool(keep_slices))
    n = hp.n
    out_ch = np.zeros(2 * (n - 1), np.int32)
    out_sl = np.zeros(len(hp.index_ids), np.int32)
    n_sl = ctypes.c_int(0)
    st = (ctypes.c_double * 8)()
    rc = lib.tnbp_optimize(n, _ptr(hp.leaf_ptr), _ptr(hp.leaf_idx), len(hp.index_ids),
                           hp.sliceable.tobytes(), _ptr(hp.init_children),
                           _ptr(init_sl) if len(init_sl) else None, len(init_sl), ctypes.byref(opt),
                           _ptr(out_ch), _ptr(out_sl), ctypes.byref(n_sl), st)
    if rc:
        msg = lib.tnbp_last_error().decode()
        if rc == 2:
            from .errors import CannotReachCap
            raise CannotReachCap(msg)
        raise ValueError(msg)
    sliced = [hp.index_ids[k] for k in out_sl[: n_sl.value]]
    new_tree = _splice_head(tree, hp, out_ch)
    plan = _plan(tn, tree, new_tree, sliced, target_space)
    if stats is not None:
        stats.update(log2_cost=st[0], sc=int(st[1]), log2_total=st[2], log2_best_unsliced=st[3],
                     trees=int(st[4]), seconds=st[5], winner=int(st[6]), plans=int(st[7]),
                     objective=objective)
    return plan, new_tree


def _splice_head(tree, hp: HeadProblem, children: np.ndarray):
    """Head steps from the SSA children; tail steps and the root step kept
    (the root step must stay last, ordering.py:164-165)."""
    Step = type(tree.steps[0])
    root = tree.steps[tree.first_cut]
    all_ids = set(tree.leaves) | {s.out for s in tree.steps}
    nxt = max(all_ids) + 1
    n = hp.n
    ids = list(hp.head_leaves)
    head = []
    for i in range(n - 1):
        out = root.lhs if i == n - 2 else nxt
        if i != n - 2:
            nxt += 1
        head.append(Step(lhs=ids[children[2 * i]], rhs=ids[children[2 * i + 1]], out=out))
        ids.append(out)
    steps = head + list(tree.tail_steps()) + [root]
    fields = {f.name for f in dataclasses.fields(tree)}
    kw = dict(steps=steps, first_cut=len(steps) - 1)
    if "annotations" in fields:
        kw["annotations"] = None
    return dataclasses.replace(tree, **kw)


def _plan(tn, old_tree, tree, sliced, target_space):
    head_leaves, _ = tree.head_tail_leaves()
    leaf_sets = {nid: frozenset(tn.nodes[nid].indices) for nid in tree.leaves}
    tc, sc = step_mults(leaf_sets, tree.head_steps(), frozenset(sliced))
    sc = max(sc, max(len(leaf_sets[h] - frozenset(sliced)) for h in head_leaves))
    base_tc, _ = step_mults(leaf_sets, old_tree.head_steps(), frozenset())
    plan = SlicePlan(
        sliced_indices=list(sliced),
        per_subtask=Complexity(tc=tc, sc_log2=sc, per_step=[]),
        overhead=((1 << len(sliced)) * tc / base_tc) if base_tc else 1.0,
        target_space=target_space,
    )
    open_ixs = frozenset(tn.open_output_indices.values())
    t_tc, t_sc = step_mults(leaf_sets, tree.tail_steps(), open_ixs)
    plan.tail_per_assignment = Complexity(tc=t_tc, sc_log2=t_sc, per_step=[])
    return plan


def plan_subtask(tn, tree, plan) -> dict:
    """The order document's ``subtask`` block (cli.py slice command format)."""
    n_e = len(plan.sliced_indices)
    tc = int(plan.per_subtask.tc)
    tail = plan.tail_per_assignment
    n_open = len(tn.open_output_indices)
    t_head = tc << n_e
    t_tail = int(tail.tc) << n_open if tail is not None else 0
    return {"count": 1 << n_e, "n_e": n_e, "overhead": plan.overhead,
            "sc_log2": int(plan.per_subtask.sc_log2), "t_head": t_head, "t_tail": t_tail,
            "t_total": t_head + t_tail, "tail_sc_log2": int(tail.sc_log2) if tail else 0,
            "tail_tc": int(tail.tc) if tail else 0, "target_space": plan.target_space, "tc": tc}


def log2(x) -> float:
    return math.log2(x) if x else float("-inf")
