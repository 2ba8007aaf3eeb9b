"""Host-side schedule helpers for the executor.

* ``split`` restates the engine's head/tail split (engine.py:171-185) and
  ``cut_indices`` (ordering.py:372-380) on duck-typed networks/trees.
* ``step_mults`` is the engine's exact multiplication counter
  (engine.py:138-140) evaluated analytically from index sets;
  ``cluster_small_steps`` re-orders a step list so the executor can batch
  its tiny steps.  (The head-absorbed tail is ordered by the native
  planner, ``treeopt.order_network``.)
"""

from __future__ import annotations


def cut_indices(tn, head: set, tail: set) -> list:
    crossing = []
    for ix, eps in tn.index_endpoints.items():
        if len(eps) == 2:
            in_head = [e in head for e in eps]
            if any(in_head) and not all(in_head):
                crossing.append(ix)
    return sorted(crossing)


def split(tn, tree):
    """(head_leaves, head_steps, tail_leaves, tail_steps, cut ids)."""
    if tree.first_cut is not None:
        head_leaves, tail_leaves = tree.head_tail_leaves()
        cut = cut_indices(tn, set(head_leaves), set(tail_leaves))
        return sorted(head_leaves), tree.head_steps(), sorted(tail_leaves), tree.tail_steps(), cut
    if tn.open_output_indices:
        return [], [], sorted(tree.leaves), list(tree.steps), []
    return sorted(tree.leaves), list(tree.steps), [], [], []


def step_mults(leaf_sets: dict, steps, removed=frozenset()) -> tuple:
    """(sum of 2^(|a|+|b|-|a&b|), max result rank) over a step list with
    `removed` indices pinned -- the engine's exact counter (engine.py:138-140)."""
    sets = {k: frozenset(v) - removed for k, v in leaf_sets.items()}
    total = 0
    rank = 0
    for s in steps:
        lhs, rhs, out = (s.lhs, s.rhs, s.out) if hasattr(s, "lhs") else s
        a, b = sets[lhs], sets[rhs]
        total += 1 << (len(a) + len(b) - len(a & b))
        sets[out] = a ^ b
        rank = max(rank, len(sets[out]))
    return total, rank


def _tiled_simt(na: int, nb: int, nab: int, tc_min_rank: int = 26) -> bool:
    """Whether the executor runs a step on the tiled SIMT kernel (the only
    kind it batches): not tensor-core eligible (program.cu tc_eligible) and
    not the streaming small-K kernel (tnb_internal.h simt_uses_smallk)."""
    tc = nab >= 3 and na + nb + nab >= tc_min_rank and max(na, nb) >= 7 and min(na, nb) >= 3
    smallk = nab <= 3 and nb >= 2 and na + nb >= 16
    return not tc and not smallk


def cluster_small_steps(leaf_sets: dict, steps, removed=frozenset()):
    """A topological re-ordering of a step list in which every step the
    executor batches (tiled SIMT) runs as soon as it is ready, all ready ones
    together, while the other steps keep their relative order.

    The executor launches consecutive independent tiled-SIMT steps as one
    kernel (program.cu plan_simt_batches); a post-order interleaves them
    with big steps and dependencies, so trees re-ordered for many small
    steps (treeopt keep_slices, slice_batch) pay one launch per tiny step.
    The result contracts the same tensors (any topological order does)."""
    sets = {k: frozenset(v) - removed for k, v in leaf_sets.items()}
    steps = list(steps)
    info = []
    for s in steps:
        lhs, rhs, out = (s.lhs, s.rhs, s.out) if hasattr(s, "lhs") else s
        a, b = sets[lhs], sets[rhs]
        sets[out] = a ^ b
        nab = len(a & b)
        info.append((lhs, rhs, out, _tiled_simt(len(a) - nab, len(b) - nab, nab)))
    produced = {o: i for i, (_, _, o, _) in enumerate(info)}
    waiting = {}
    ndeps = []
    for i, (l, r, _, _) in enumerate(info):
        deps = [produced[x] for x in (l, r) if x in produced]
        ndeps.append(len(deps))
        for d in deps:
            waiting.setdefault(d, []).append(i)
    import heapq

    ready_small = [i for i, n in enumerate(ndeps) if n == 0 and info[i][3]]
    ready_big = [i for i, n in enumerate(ndeps) if n == 0 and not info[i][3]]
    heapq.heapify(ready_small)
    heapq.heapify(ready_big)
    order = []

    def done(i):
        order.append(i)
        for j in waiting.get(i, ()):
            ndeps[j] -= 1
            if ndeps[j] == 0:
                heapq.heappush(ready_small if info[j][3] else ready_big, j)

    while ready_small or ready_big:
        if ready_small:
            batch = []
            while ready_small:
                batch.append(heapq.heappop(ready_small))
            for i in batch:  # one wave of mutually independent small steps
                done(i)
        else:
            done(heapq.heappop(ready_big))
    if len(order) != len(steps):
        raise ValueError("step list is not a valid pairwise order")
    return [steps[i] for i in order]
