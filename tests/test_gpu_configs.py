"""Further BASELINE configs on the GPU: C3 (m=14, 2^16 bitstrings, t=2^30) and
the C5 sweep points t=2^26 (n_e=63), t=2^28 (n_e=58), 2^21 bitstrings, and
t=2^32 (fused vs staged) -- needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2, measured
from oracle import engine_np as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.mark.parametrize("name,rng_", [("c3", (0, 1)), ("c5_26", (0, 2)), ("c5_28", (0, 1)),
                                       ("c5_n21", (0, 1))])
def test_config_head_tail_xeb_vs_reference(gpu, workloads, name, rng_):
    w = workloads(name)
    g = golden(name)
    a, b = rng_
    st = tnb.EngineStats()
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=rng_,
                                 precision="single", stats=st)
    key = f"head_single_{a}_{b}"
    stride = int(g["stride"])
    assert measured(rel_l2(hv.data[::stride], g[key + "_sub"])) < TOL
    assert abs(float(np.vdot(hv.data, hv.data).real) / float(g[key + "_norm2"]) - 1) < 2 * TOL
    # exact reference counters (engine.py:138-140)
    assert [st.multiplications, st.head_contractions] == [int(g[key + "_stats"][0]),
                                                          int(g[key + "_stats"][1])]
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    s2 = int(g["amps_stride"])
    assert measured(rel_l2(tab.amplitudes[::s2], g["amps_sub"])) < TOL
    probs = np.abs(tab.amplitudes.astype(np.complex128)) ** 2
    f_ref = (2.0 ** 53 / probs.size) * float(g["amps_probsum"]) - 1.0
    assert measured(abs(O.xeb(probs, 53) - f_ref), 'xeb_abs') < 1e-3


def test_n_e_63_mask_bits(gpu, workloads):
    """63 sliced edges: masks near 2^63 address the top mask bits correctly."""
    w = workloads("c5_26")
    assert w.n_e == 63
    top = (1 << 63) - 2
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(top, top + 2),
                                 precision="single")
    assert hv.slice_range == (top, top + 2)
    assert np.isfinite(hv.data).all() and np.abs(hv.data).max() > 0


def test_c5_32_fused_matches_staged(gpu, workloads):
    """t = 2^32 (n_e = 48): intermediates of 2^32 elements, whose fused
    operands use the full 32-bit destination index range.  No reference
    golden exists at this size (one CPU slice takes minutes), so the fused
    program is checked against the staged one (TNB_FLAG_NO_FUSE), which the
    other configs pin to the reference."""
    import gc

    from paper_2103_03074_b200 import _lib, engine as E

    w = workloads("c5_32")
    E.clear_cache()
    fused = E.head_program(w.tn, w.tree, w.sliced, "single", flags=0)
    assert fused.info.n_steps_fused > 0
    hf = fused.run_range(0, 1)
    del fused
    E.clear_cache()
    gc.collect()
    staged = E.head_program(w.tn, w.tree, w.sliced, "single", flags=_lib.TNB_FLAG_NO_FUSE)
    hs = staged.run_range(0, 1)
    del staged
    E.clear_cache()
    gc.collect()
    assert np.isfinite(hf).all() and np.abs(hs).max() > 0
    assert measured(rel_l2(hf, hs)) < 1e-5
