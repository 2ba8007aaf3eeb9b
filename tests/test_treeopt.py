"""Head-tree / slice co-optimiser -- CPU tests.

The frozen co-optimised plans (tests/golden/*_opt, made by
make_opt_plans.py) must be valid drop-ins for the reference planner's:
same leaves, head leaves, cut legs, tail and root step; sliced indices
head-internal; space target met; the document's subtask figures exact.
Their results are pinned by the reference engine's own goldens
(make_goldens.py) -- here through the oracle, on the GPU in
test_gpu_treeopt.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, import_reference, reference_available, rel_l2
from paper_2103_03074_b200 import treeopt
from paper_2103_03074_b200.planner import split, step_mults

OPT = {"c1_opt": "c1", "s8_opt": "s8", "c4_opt": "c4", "c4_opt_b200": "c4", "c4_reordered": "c4",
       "c4_opt31": "c4", "c4_opt31_b200": "c4", "c2_opt_b200": "c2", "c2_opt_b200_alt": "c2", "c3_opt_b200": "c3",
       "c3_opt_b200_alt": "c3",
       "c5_26_reordered": "c5_26", "c5_28_reordered": "c5_28", "c5_32_reordered": "c5_32"}


@pytest.fixture(scope="module")
def lib():
    treeopt.build()
    return treeopt.load()


def test_plan_lib_exports_header_symbols(lib):
    with open(os.path.join(ROOT, "include", "tnb_plan.h")) as fh:
        declared = set(re.findall(r"\b(tnbp_\w+)\s*\(", fh.read()))
    assert declared == set(treeopt.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym


@pytest.mark.parametrize("name", sorted(OPT))
def test_frozen_plan_is_a_drop_in(workloads, name):
    w, base = workloads(name), workloads(OPT[name])
    assert sorted(w.tree.leaves) == sorted(base.tree.leaves)
    assert w.tree.first_cut == len(w.tree.steps) - 1  # ordering.py:164-165
    assert w.tree.steps[-1] == base.tree.steps[base.tree.first_cut]
    hl, hs, tl, ts, cut = split(w.tn, w.tree)
    bhl, _, btl, bts, bcut = split(base.tn, base.tree)
    assert (hl, tl, ts, cut) == (bhl, btl, bts, bcut)
    # a valid pairwise tree over the head leaves (validate_tree semantics)
    avail = set(hl)
    for s in hs:
        assert s.lhs in avail and s.rhs in avail and s.out not in avail
        avail -= {s.lhs, s.rhs}
        avail.add(s.out)
    assert avail == {w.tree.steps[-1].lhs}
    # sliced indices are head-internal bonds (slicing.py:97-102)
    hset = set(hl)
    for ix in w.sliced:
        eps = w.tn.index_endpoints[ix]
        assert len(eps) == 2 and set(eps) <= hset
    # exact subtask figures (engine.py:138-140 counter) and the space target
    sets = {nid: frozenset(w.tn.nodes[nid].indices) for nid in w.tree.leaves}
    tc, sc = step_mults(sets, hs, frozenset(w.sliced))
    assert tc == w.tc_per_slice and sc <= w.target_space
    # strictly less total head work than the reference plan
    assert math.log2(tc) + w.n_e < math.log2(base.tc_per_slice) + base.n_e
    assert w.doc["planner"]["log2_total_work_saved"] > 0


def test_c1_opt_full_sum_is_plan_independent(workloads):
    """All slices of the co-optimised plan sum to the reference plan's head
    vector and to the state vector's amplitudes (oracle, double)."""
    from oracle import engine_np as O

    w = workloads("c1_opt")
    g1, g = golden("c1"), golden("c1_opt")
    hv = O.head_vector(w.tn, w.tree, w.sliced, None, "double")
    assert np.abs(hv - g1["head_full_double"]).max() < 1e-12
    assert np.abs(hv - g["head_full_double"]).max() < 1e-12
    amps = O.tail_absorbed(w.tn, w.tree, hv, "double")
    assert np.abs(amps - g1["amps_statevector"][0]).max() < 1e-12


def test_s8_opt_oracle_matches_reference_goldens(workloads):
    from oracle import engine_np as O

    w, g = workloads("s8_opt"), golden("s8_opt")
    hv = O.head_vector(w.tn, w.tree, w.sliced, (0, 4), "double")
    stride = int(g["stride"])
    assert rel_l2(hv[::stride], g["head_double_0_4_sub"]) < 1e-10


def test_optimiser_deterministic_and_never_worse(workloads, lib):
    w = workloads("s8")
    kw = dict(trials=64, keep_top=4, reconf_k=8, polish_k=8, time_budget_s=600, seed=3,
              initial_slices=w.sliced)
    p1, t1 = treeopt.select_slices_b200(w.tn, w.tree, w.target_space, threads=1, **kw)
    p2, t2 = treeopt.select_slices_b200(w.tn, w.tree, w.target_space, threads=4, **kw)
    assert p1.sliced_indices == p2.sliced_indices and t1.steps == t2.steps
    ref_total = math.log2(w.tc_per_slice) + w.n_e
    assert math.log2(p1.per_subtask.tc) + len(p1.sliced_indices) <= ref_total
    assert p1.per_subtask.sc_log2 <= w.target_space
    # the b200 objective re-ranks candidates by the time model and polishes
    # the winner under it: never slower (in the model) than the mults plan
    pb, tb = treeopt.select_slices_b200(w.tn, w.tree, w.target_space, objective="b200", **kw)
    assert (treeopt.tree_cost(w.tn, tb, pb.sliced_indices, "b200")[2]
            <= treeopt.tree_cost(w.tn, t1, p1.sliced_indices, "b200")[2] + 1e-9)


def test_b200_polish_keeps_slices_and_lowers_model_time(workloads, lib):
    """c4_opt_b200 = c4_opt's sliced set, subtrees re-optimised under the
    B200 time model (merging small operands before they meet a big one)."""
    w, b = workloads("c4_opt"), workloads("c4_opt_b200")
    assert b.sliced == w.sliced
    assert (treeopt.tree_cost(b.tn, b.tree, b.sliced, "b200")[0]
            < treeopt.tree_cost(w.tn, w.tree, w.sliced, "b200")[0] - 0.2)


def test_reordered_keeps_the_reference_slices(workloads, lib):
    w, r = workloads("c4_reordered"), workloads("c4")
    assert w.sliced == r.sliced
    assert math.log2(w.tc_per_slice) < math.log2(r.tc_per_slice) - 4


def test_restarts_keep_the_best_seed(workloads, lib):
    w = workloads("s8")
    kw = dict(trials=16, keep_top=2, reconf_k=6, polish_k=6, time_budget_s=600, threads=2)
    totals = []
    for sd in (5, 6):
        st = {}
        treeopt.select_slices_b200(w.tn, w.tree, w.target_space, seed=sd, stats=st, **kw)
        totals.append(st["log2_total"])
    st = {}
    treeopt.select_slices_b200(w.tn, w.tree, w.target_space, seed=5, restarts=2, stats=st, **kw)
    assert abs(st["log2_total"] - min(totals)) < 1e-9 and st["restarts"] == 2


def test_unreachable_target_raises(workloads, lib):
    from paper_2103_03074_b200.errors import CannotReachCap

    w = workloads("c1")
    with pytest.raises(CannotReachCap):
        # the cut legs (n_c = 5) cannot be sliced
        treeopt.select_slices_b200(w.tn, w.tree, 4, trials=8, keep_top=2)


def test_bad_input_is_an_error(lib):
    opt = treeopt.Options()
    lib.tnbp_default_options(ctypes.byref(opt))
    ptr = np.array([0, 1, 2, 3], np.int32)
    idx = np.array([0, 0, 0], np.int32)  # one index on three leaves
    out = np.zeros(4, np.int32)
    st = (ctypes.c_double * 8)()
    n = ctypes.c_int(0)
    rc = lib.tnbp_optimize(3, treeopt._ptr(ptr), treeopt._ptr(idx), 1, b"\x01", None, None, 0,
                           ctypes.byref(opt), treeopt._ptr(out), treeopt._ptr(out),
                           ctypes.byref(n), st)
    assert rc == 1 and b"endpoints" in lib.tnbp_last_error()


@pytest.mark.skipif(not reference_available(), reason="reference package not present")
def test_reference_accepts_the_plan(workloads):
    """The reference's own validate_tree / complexity_of / doc loader take
    the frozen co-optimised order document."""
    import json

    import_reference()
    from tncut import ordering as tord

    w = workloads("s8_opt")
    with open(os.path.join(ROOT, "tests", "golden", "s8_opt", "order.json")) as fh:
        tree = tord.doc_to_tree(json.load(fh))
    assert tree.first_cut == len(tree.steps) - 1
    assert [(s.lhs, s.rhs, s.out) for s in tree.steps] == [(s.lhs, s.rhs, s.out) for s in w.tree.steps]


def test_keep_slices_argument_checks(workloads, lib):
    from paper_2103_03074_b200.errors import ShapeMismatch

    w = workloads("s8")
    with pytest.raises(ValueError):
        treeopt.select_slices_b200(w.tn, w.tree, w.target_space, keep_slices=True)
    with pytest.raises(ShapeMismatch):
        treeopt.select_slices_b200(w.tn, w.tree, w.target_space, keep_slices=True,
                                   initial_slices=[10 ** 9])
    plan, tree = treeopt.select_slices_b200(w.tn, w.tree, w.target_space, keep_slices=True,
                                            initial_slices=w.sliced)
    assert plan.sliced_indices == w.sliced
    assert plan.per_subtask.tc <= w.tc_per_slice
