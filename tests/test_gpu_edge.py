"""Edge cases of the device path -- needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2
from oracle import engine_np as O

pytestmark = pytest.mark.gpu


def test_unsliced_head_single_range(gpu, workloads):
    """n_e = 0: one 'slice' (the whole head), mask range [0, 1)."""
    w = workloads("c1")
    hv = tnb.compute_head_vector(w.tn, w.tree, [], None, precision="double")
    ref = O.head_vector(w.tn, w.tree, [], precision="double")
    assert hv.n_e == 0 and hv.slice_range == (0, 1)
    assert rel_l2(hv.data, ref) < 1e-12
    # the unsliced head equals the sum over all slices of the sliced plan
    sliced = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="double")
    assert rel_l2(hv.data, sliced.data) < 1e-12


def test_m12_double_precision_tensor_sized_steps(gpu, workloads):
    """fp64 SIMT path on a plan whose big steps use tcgen05 in single precision."""
    w = workloads("m12")
    g = golden("m12")
    if "head_double_0_1_sub" not in g:
        pytest.skip("double golden not generated")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 1),
                                 precision="double")
    stride = int(g["stride"])
    assert rel_l2(hv.data[::stride], g["head_double_0_1_sub"]) < 1e-10


def test_free_mode_long_range_matches_fixed(gpu, workloads):
    """free (running sum) vs fixed (binary tree) over 64 slices agree to fp rounding."""
    w = workloads("s8")
    a = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 64),
                                precision="single", mode="fixed")
    b = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 64),
                                precision="single", mode="free")
    assert rel_l2(a.data, b.data) < 1e-5  # summation orders differ; values agree


def test_repin_changes_leaves_only(gpu, workloads):
    """A new s1 reuses the compiled program (same topology) and matches the oracle."""
    w = workloads("s8")
    s1 = "".join("1" if i % 3 == 0 else "0" for i in range(len(w.tn.fixed_output_bits)))
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s1, slice_range=(0, 2),
                                 precision="single")
    bits = {q: int(b) for q, b in zip(sorted(w.tn.fixed_output_bits), s1)}
    ref = O.head_vector(w.tn.repin(bits), w.tree, w.sliced, (0, 2), "single")
    assert rel_l2(hv.data, ref) < 1e-4
    assert hv.s1 == bits
