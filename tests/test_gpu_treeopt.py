"""Co-optimised plans (treeopt) on the GPU executor.

The plans in tests/golden/*_opt keep the reference's network, head/tail
partition and cut; their goldens come from the unmodified reference engine
run on the SAME plans (make_goldens.py).  c1_opt additionally checks the
plan-independence of the full slice sum against c1 and the state vector.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2, measured
from oracle import engine_np as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.mark.parametrize("precision,tol", [("double", 1e-10), ("single", TOL)])
def test_c1_opt_full_sum_equals_reference_plan_and_statevector(gpu, workloads, precision, tol):
    w = workloads("c1_opt")
    g1, g = golden("c1"), golden("c1_opt")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision=precision)
    assert measured(rel_l2(hv.data, g["head_full_double"])) < tol
    assert measured(rel_l2(hv.data, g1["head_full_double"])) < tol
    tab = tnb.compute_tail_amplitudes(w.tn, w.tree, hv, precision=precision)
    assert measured(rel_l2(tab.amplitudes, g1["amps_statevector"][0])) < tol
    for a, b in [(0, 1), (1, 4)]:
        p = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(a, b),
                                    precision=precision)
        assert measured(rel_l2(p.data, g[f"head_fixed_{a}_{b}"])) < tol


@pytest.mark.parametrize("name,rng_", [("s8_opt", (0, 4)), ("s8_opt", (0, 1)), ("c4_opt", (0, 1)),
                                       ("c4_opt_b200", (0, 1)), ("c4_opt31_b200", (0, 1)),
                                       ("c2_opt_b200", (0, 1)), ("c3_opt_b200", (0, 1))])
def test_opt_plan_head_tail_xeb_vs_reference(gpu, workloads, name, rng_):
    w, g = workloads(name), golden(name)
    a, b = rng_
    st = tnb.EngineStats()
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=rng_,
                                 precision="single", stats=st)
    key = f"head_single_{a}_{b}"
    stride = int(g["stride"])
    assert measured(rel_l2(hv.data[::stride], g[key + "_sub"])) < TOL
    assert abs(float(np.vdot(hv.data, hv.data).real) / float(g[key + "_norm2"]) - 1) < 2 * TOL
    assert [st.multiplications, st.head_contractions] == [int(g[key + "_stats"][0]),
                                                          int(g[key + "_stats"][1])]
    if (a, b) != (0, 1) or name[:2] in ("c2", "c3", "c4"):
        tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
        s2 = int(g["amps_stride"])
        assert measured(rel_l2(tab.amplitudes[::s2], g["amps_sub"])) < TOL
        probs = np.abs(tab.amplitudes.astype(np.complex128)) ** 2
        f_ref = (2.0 ** 53 / probs.size) * float(g["amps_probsum"]) - 1.0
        assert measured(abs(O.xeb(probs, 53) - f_ref), 'xeb_abs') < 1e-3


def test_c4_reordered_same_slices_as_reference_plan(gpu, workloads):
    """c4_reordered keeps the reference plan's sliced set (same masks, same
    partial head vectors) with a re-ordered head tree: its slice [0,1)
    equals the reference engine's c4 golden; slices [0,4) equal the
    executor's own result on the reference tree."""
    w, r = workloads("c4_reordered"), workloads("c4")
    assert w.sliced == r.sliced
    g = golden("c4")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 1), precision="single")
    stride = int(g["stride"])
    assert measured(rel_l2(hv.data[::stride], g["head_single_0_1_sub"])) < TOL
    a = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 4), precision="single")
    b = tnb.compute_head_vector(r.tn, r.tree, r.sliced, None, slice_range=(0, 4), precision="single")
    assert measured(rel_l2(a.data, b.data)) < TOL


def test_set_reorder_same_head_vectors(gpu, workloads):
    """Opt-in re-ordering through the public API: same slices, same partial
    head vectors (vs the reference goldens), reference counters unchanged."""
    from paper_2103_03074_b200 import engine as E

    try:
        tnb.set_reorder(True)
        for name, rng_ in (("s8", (0, 4)), ("c4", (0, 1))):
            w, g = workloads(name), golden(name)
            st = tnb.EngineStats()
            hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=rng_,
                                         precision="single", stats=st)
            key = f"head_single_{rng_[0]}_{rng_[1]}"
            assert measured(rel_l2(hv.data[::int(g["stride"])], g[key + "_sub"])) < TOL
            assert [st.multiplications, st.head_contractions] == [int(g[key + "_stats"][0]),
                                                                  int(g[key + "_stats"][1])]
        assert len(E._reorder_cache) >= 2
    finally:
        tnb.set_reorder(False)


@pytest.mark.parametrize("name,rng_", [("c5_26", (0, 2)), ("c5_28", (0, 1))])
def test_sweep_reordered_same_slices_vs_reference(gpu, workloads, name, rng_):
    w, g = workloads(name + "_reordered"), golden(name)
    assert w.sliced == workloads(name).sliced
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=rng_, precision="single")
    key = f"head_single_{rng_[0]}_{rng_[1]}"
    assert measured(rel_l2(hv.data[::int(g["stride"])], g[key + "_sub"])) < TOL


def test_c5_32_reordered_matches_given_tree(gpu, workloads):
    import gc

    w, r = workloads("c5_32_reordered"), workloads("c5_32")
    a = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 1), precision="single")
    tnb.clear_cache()
    gc.collect()
    b = tnb.compute_head_vector(r.tn, r.tree, r.sliced, None, slice_range=(0, 1), precision="single")
    tnb.clear_cache()
    assert measured(rel_l2(a.data, b.data)) < TOL


def test_c2_complete_contraction_is_plan_independent(gpu, workloads):
    """ALL slices of two independently co-optimised C2 plans (different
    trees and sliced sets): the complete head sums give the same 2^10
    amplitudes and XEB (a finished 53-qubit m=12 answer, ~1 min)."""
    import gc

    amps = []
    try:
        tnb.set_slice_batch(3)
        for name in ("c2_opt_b200", "c2_opt_b200_alt"):
            w = workloads(name)
            hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="single")
            assert hv.slice_range == (0, 1 << w.n_e)
            tab = tnb.compute_tail_amplitudes(w.tn, w.tree, hv, precision="single")
            amps.append(tab.amplitudes.astype(np.complex128))
            tnb.clear_cache()
            gc.collect()
    finally:
        tnb.set_slice_batch(0)
    assert measured(rel_l2(amps[1], amps[0])) < TOL
    p0, p1 = np.abs(amps[0]) ** 2, np.abs(amps[1]) ** 2
    assert abs(O.xeb(p0, 53) - O.xeb(p1, 53)) < 1e-3
