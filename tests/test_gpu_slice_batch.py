"""Batched slices (slice_batch.py): 2^k aligned slices
per contraction by un-slicing the lowest-mask-bit sliced indices."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2, measured
from paper_2103_03074_b200.slice_batch import compute_head_vector_slice_batched as batched

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.mark.parametrize("reorder", [False, True])
def test_s8_blocks_match_reference_goldens(gpu, workloads, reorder):
    w, g = workloads("s8"), golden("s8")
    stride = int(g["stride"])
    parts = []
    for a, b in [(0, 4), (4, 8)]:
        st = tnb.EngineStats()
        hv = batched(w.tn, w.tree, w.sliced, None, slice_range=(a, b), batch_log2=2,
                     reorder=reorder, stats=st)
        key = f"head_single_{a}_{b}"
        assert measured(rel_l2(hv.data[::stride], g[key + "_sub"])) < TOL
        assert [st.multiplications, st.head_contractions] == [int(g[key + "_stats"][0]),
                                                              int(g[key + "_stats"][1])]
        assert hv.slice_range == (a, b) and hv.n_e == w.n_e
        parts.append(hv)
    # aligned 2^k partials recombine bit-exactly with the one-call result
    # (the binary-counter merge of two blocks is block0 + block1,
    # engine.py:207-222; reduce_partials itself needs full coverage)
    whole = batched(w.tn, w.tree, w.sliced, None, slice_range=(0, 8), batch_log2=2, reorder=reorder)
    assert np.array_equal(parts[0].data + parts[1].data, whole.data)
    assert parts[0].provenance == whole.provenance


def test_c4_block_matches_per_slice_path(gpu, workloads):
    w = workloads("c4")
    hv = batched(w.tn, w.tree, w.sliced, None, slice_range=(0, 16), batch_log2=4)
    ref = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 16),
                                  precision="single")
    assert measured(rel_l2(hv.data, ref.data)) < TOL
    assert hv.provenance == ref.provenance
    tnb.clear_cache()


def test_misaligned_range_raises(gpu, workloads):
    w = workloads("s8")
    with pytest.raises(tnb.RangeOutOfBounds):
        batched(w.tn, w.tree, w.sliced, None, slice_range=(2, 6), batch_log2=2)


def test_public_api_opt_in(gpu, workloads):
    w = workloads("c4")
    ref = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(16, 32),
                                  precision="single")
    try:
        tnb.set_slice_batch(4)
        st = tnb.EngineStats()
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(16, 32),
                                     precision="single", stats=st)
        odd = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(16, 18),
                                      precision="single")  # unaligned: per-slice path
    finally:
        tnb.set_slice_batch(0)
    assert measured(rel_l2(hv.data, ref.data)) < TOL
    assert st.head_contractions == 16 and st.multiplications == 16 * w.tc_per_slice
    assert odd.slice_range == (16, 18)
    tnb.clear_cache()


def test_co_optimised_plan_blocks_match_per_slice(gpu, workloads):
    """Batching on top of the co-optimised plan (rank-32 intermediates)."""
    import gc

    w = workloads("c4_opt31_b200")
    hv = batched(w.tn, w.tree, w.sliced, None, slice_range=(0, 4), batch_log2=2, max_rank=32)
    tnb.clear_cache()
    gc.collect()
    ref = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 4),
                                  precision="single")
    tnb.clear_cache()
    assert measured(rel_l2(hv.data, ref.data)) < TOL


def test_public_api_falls_back_to_narrower_blocks(gpu, workloads):
    """C5_32 (rank-32 plan): 2^4 blocks would need rank > 32, so the API
    takes the widest block that fits (or the per-slice path) silently."""
    import gc

    w = workloads("c5_32")
    try:
        tnb.set_slice_batch(4)
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 16),
                                     precision="single")
    finally:
        tnb.set_slice_batch(0)
    tnb.clear_cache()
    gc.collect()
    assert hv.slice_range == (0, 16) and np.isfinite(hv.data).all()
