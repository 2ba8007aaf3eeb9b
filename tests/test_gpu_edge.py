"""Edge cases of the device path -- needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2, measured
from oracle import engine_np as O

pytestmark = pytest.mark.gpu


def test_unsliced_head_single_range(gpu, workloads):
    """n_e = 0: one 'slice' (the whole head), mask range [0, 1)."""
    w = workloads("c1")
    hv = tnb.compute_head_vector(w.tn, w.tree, [], None, precision="double")
    ref = O.head_vector(w.tn, w.tree, [], precision="double")
    assert hv.n_e == 0 and hv.slice_range == (0, 1)
    assert measured(rel_l2(hv.data, ref)) < 1e-12
    # the unsliced head equals the sum over all slices of the sliced plan
    sliced = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="double")
    assert measured(rel_l2(hv.data, sliced.data)) < 1e-12


def test_m12_double_precision_tensor_sized_steps(gpu, workloads):
    """fp64 SIMT path on a plan whose big steps use tcgen05 in single precision."""
    w = workloads("m12")
    g = golden("m12")
    if "head_double_0_1_sub" not in g:
        pytest.skip("double golden not generated")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 1),
                                 precision="double")
    stride = int(g["stride"])
    assert measured(rel_l2(hv.data[::stride], g["head_double_0_1_sub"])) < 1e-10


def test_free_mode_long_range_matches_fixed(gpu, workloads):
    """free (running sum) vs fixed (binary tree) over 64 slices agree to fp rounding."""
    w = workloads("s8")
    a = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 64),
                                precision="single", mode="fixed")
    b = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 64),
                                precision="single", mode="free")
    assert measured(rel_l2(a.data, b.data)) < 1e-5  # summation orders differ; values agree


def test_repin_changes_leaves_only(gpu, workloads):
    """A new s1 reuses the compiled program (same topology) and matches the oracle."""
    w = workloads("s8")
    s1 = "".join("1" if i % 3 == 0 else "0" for i in range(len(w.tn.fixed_output_bits)))
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s1, slice_range=(0, 2),
                                 precision="single")
    bits = {q: int(b) for q, b in zip(sorted(w.tn.fixed_output_bits), s1)}
    ref = O.head_vector(w.tn.repin(bits), w.tree, w.sliced, (0, 2), "single")
    assert measured(rel_l2(hv.data, ref)) < 1e-4
    assert hv.s1 == bits


@pytest.mark.parametrize("name,precision", [("c2", "single"), ("s8", "double")])
def test_tail_space_cap_blocks_the_open_qubits(gpu, workloads, name, precision):
    """space_cap below the absorbed tail's largest intermediate: the k leading
    open qubits are pinned (engine.py:348-362) and the 2^k blocks fill the
    amplitude vector in s2 order -- same amplitudes as the one-block tail."""
    from paper_2103_03074_b200 import engine as E
    from paper_2103_03074_b200.planner import step_mults

    w = workloads(name)
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 2),
                                 precision=precision)
    full = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision=precision)
    tn = w.tn.repin(hv.s1)
    leaves, hid, steps = E.tail_plan(tn, w.tree, hv.cut_order)
    sets = {nid: tn.nodes[nid].indices for nid in leaves}
    sets[hid] = list(hv.cut_order)
    opens = [tn.open_output_indices[q] for q in sorted(tn.open_output_indices)]
    r0 = step_mults(sets, steps)[1]
    cap = r0 - 2
    k = 0
    while k < len(opens) and step_mults(sets, steps, frozenset(opens[:k]))[1] > cap:
        k += 1
    assert 1 <= k < len(opens), (r0, k)
    blocked = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, space_cap=cap, precision=precision)
    tol = 1e-6 if precision == "single" else 1e-12
    assert measured(rel_l2(blocked.amplitudes, full.amplitudes)) < tol
    assert blocked.amplitudes.dtype == full.amplitudes.dtype
