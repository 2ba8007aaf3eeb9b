"""Batched slices (second half): 2^k consecutive slices
of an aligned block contracted in ONE pass by un-slicing the k sliced
indices that carry the lowest mask bits.

The engine's mask convention pins ``sliced[pos]`` to mask bit
``n_e-1-pos`` (engine.py:276-279), so the masks of an aligned block
``[j*2^k, (j+1)*2^k)`` differ exactly in ``sliced[-k:]``.  Summing a head
contraction over both values of a sliced index is contracting that index
(slicing.py:1-12), so one contraction of the plan with ``sliced[:-k]``
yields the block's sum of partial head vectors: the slice units and the
result of ``compute_head_vector(slice_range=(a, b))`` stay the same, the
GEMMs get 2^k times more work per launch and the per-slice launch and
staging overheads shrink by 2^k.  With ``reorder`` the head tree is
re-ordered for the reduced sliced set (``treeopt`` keep_slices, exact DP +
B200 polish), since un-slicing changes which order is cheap.

Summation order: blocks are combined by the executor's fixed binary-counter
sum (engine.py:207-222); inside a block the 2^k terms are summed by the
contraction itself.  Results equal the per-slice path within fp32
rounding, and partials of ranges aligned to 2^k recombine bit-exactly
through ``reduce_partials`` (ranges finer than a block are not produced
here: ``slice_range`` must be 2^k-aligned).
"""

from __future__ import annotations

import hashlib
import os

from . import engine as E
from .errors import BlockTooWide, RangeOutOfBounds, ShapeMismatch
from .planner import cluster_small_steps, step_mults
from .provenance import normalize_s1, provenance_hash
from .types import HeadVector

_plans: dict = {}


def batched_plan(tn, tree, sliced_indices, k: int, reorder: bool = True, max_rank: int | None = None):
    """(head steps, reduced sliced set, max rank) for k un-sliced indices."""
    head_leaves, head_steps, _, _, _ = E._split(tn, tree)
    sliced = list(sliced_indices)
    if not 0 <= k <= len(sliced):
        raise ValueError(f"batch_log2 {k} outside [0, n_e={len(sliced)}]")
    reduced = sliced[: len(sliced) - k]
    key = hashlib.sha256(repr((tuple((n, tuple(tn.nodes[n].indices)) for n in head_leaves),
                               tuple(E._steps_tuples(head_steps)), tuple(sliced), k, reorder,
                               max_rank, os.environ.get("TNB_CLUSTER", "1"))).encode()).hexdigest()
    hit = _plans.get(key)
    if isinstance(hit, BlockTooWide):  # negative results are memoised too
        raise hit
    if hit is not None:
        return hit
    sets = {n: tn.nodes[n].indices for n in head_leaves}
    steps = head_steps
    if reorder and head_steps and tree.first_cut is not None:
        from . import treeopt

        _, sc0 = step_mults(sets, head_steps, frozenset(sliced))
        cap = max_rank if max_rank is not None else sc0 + k
        plan, new_tree = treeopt.select_slices_b200(tn, tree, cap, objective="b200",
                                                    keep_slices=True, initial_slices=reduced)
        if list(plan.sliced_indices) != reduced:
            raise ShapeMismatch("re-ordering changed the sliced set")
        steps = new_tree.head_steps()
    if os.environ.get("TNB_CLUSTER", "1") != "0":
        steps = cluster_small_steps(sets, steps, frozenset(reduced))
    _, sc = step_mults(sets, steps, frozenset(reduced))
    sc = max([sc] + [len(set(tn.nodes[n].indices) - set(reduced)) for n in head_leaves])
    if sc > 32:
        _plans[key] = BlockTooWide(f"un-slicing {k} indices needs rank-{sc} intermediates (> 32)")
        raise _plans[key]
    _plans[key] = (steps, reduced, sc)
    return _plans[key]


def compute_head_vector_slice_batched(tn, tree, sliced_indices, s1, slice_range=None,
                                      batch_log2: int = 3, precision: str = "single",
                                      mode: str = "fixed", stats=None, device=None,
                                      reorder: bool = True, max_rank: int | None = None) -> HeadVector:
    """``compute_head_vector`` (engine.py:242-310) over 2^batch_log2-slice blocks.

    Same arguments and result (slice units, ``HeadVector`` fields,
    provenance, reference ``EngineStats`` counters of the given tree);
    ``slice_range`` must be aligned to 2^batch_log2.
    """
    s1 = normalize_s1(tn, s1)
    tn = tn.repin(s1)
    sliced = list(sliced_indices)
    n_e = len(sliced)
    k = int(batch_log2)
    total = 1 << n_e
    a, b = slice_range if slice_range is not None else (0, total)
    if not (0 <= a < b <= total):
        raise RangeOutOfBounds(f"range [{a},{b}) outside [0,{total})")
    if a % (1 << k) or b % (1 << k):
        raise RangeOutOfBounds(f"range [{a},{b}) is not aligned to 2^{k}-slice blocks")
    if mode not in E._MODES:
        raise ValueError(f"unknown reduction mode {mode!r}")
    head_leaves, head_steps, _, _, cut = E._split(tn, tree)
    hs = set(head_leaves)
    for ix in sliced:
        eps = tn.index_endpoints.get(ix, ())
        if len(eps) != 2 or any(e not in hs for e in eps):
            raise ShapeMismatch(f"sliced index {ix} is not internal to the head")
    steps, reduced, _ = batched_plan(tn, tree, sliced, k, reorder, max_rank)
    entries = E._leaf_entries(tn, head_leaves)
    prog = E.get_program(entries, E._steps_tuples(steps), reduced, sorted(cut), precision, device,
                         upload=False)
    data = prog.run(entries, a >> k, b >> k, mode)
    if stats is not None:
        sets = {n: tn.nodes[n].indices for n in head_leaves}
        mults, _ = step_mults(sets, head_steps, frozenset(sliced))
        stats.head_contractions += b - a
        stats.multiplications += mults * (b - a)
        stats.steps_executed += len(head_steps) * (b - a)
    return HeadVector(s1=s1, data=data,
                      provenance=provenance_hash(tn, tree, s1, precision, mode, sliced),
                      cut_order=sorted(cut), n_e=n_e, slice_range=(a, b), mode=mode,
                      sliced_indices=tuple(sliced))


def batched_program(tn, tree, sliced_indices, k: int, precision="single", device=None,
                    reorder: bool = True, max_rank: int | None = None):
    """The compiled program of the batched plan (benchmarks)."""
    head_leaves, _, _, _, cut = E._split(tn, tree)
    steps, reduced, _ = batched_plan(tn, tree, sliced_indices, k, reorder, max_rank)
    return E.get_program(E._leaf_entries(tn, head_leaves), E._steps_tuples(steps), reduced,
                         sorted(cut), precision, device)
