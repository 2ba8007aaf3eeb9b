"""Batched-slice planning (slice_batch.batched_plan) -- CPU, no device."""

from __future__ import annotations

import math

import pytest

from paper_2103_03074_b200 import slice_batch as SB
from paper_2103_03074_b200 import treeopt
from paper_2103_03074_b200.planner import split, step_mults


@pytest.fixture(scope="module", autouse=True)
def _lib():
    treeopt.build()


@pytest.mark.parametrize("name,k", [("s8", 2), ("c4", 4)])
def test_batched_plan_unslices_the_lowest_mask_bits(workloads, name, k):
    w = workloads(name)
    steps, reduced, sc = SB.batched_plan(w.tn, w.tree, w.sliced, k)
    # engine.py:276-279: sliced[pos] <-> mask bit n_e-1-pos, so the k lowest
    # mask bits are the LAST k sliced indices
    assert reduced == w.sliced[: w.n_e - k]
    hl, hs, _, _, _ = split(w.tn, w.tree)
    # a valid pairwise tree over the same head leaves, ending in the head root
    avail = set(hl)
    for s in steps:
        assert s.lhs in avail and s.rhs in avail and s.out not in avail
        avail -= {s.lhs, s.rhs}
        avail.add(s.out)
    assert avail == {hs[-1].out}
    sets = {n: w.tn.nodes[n].indices for n in hl}
    mults, rank = step_mults(sets, steps, frozenset(reduced))
    assert rank <= sc <= 32
    # a block of 2^k slices costs less than 2^k slices of the given tree
    assert math.log2(mults) < math.log2(w.tc_per_slice) + k


def test_batch_too_wide_is_refused(workloads):
    w = workloads("s8")
    with pytest.raises(ValueError):
        SB.batched_plan(w.tn, w.tree, w.sliced, w.n_e + 1)
