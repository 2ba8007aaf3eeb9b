"""Batched closed-bit assignments: the un-pinned network
reproduces every repinned network (CPU), and one batched contraction gives the
per-s1 head vectors and amplitudes (GPU)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2


def _s1_list(tn, qubits):
    closed = sorted(tn.fixed_output_bits)
    base = dict(tn.fixed_output_bits)
    out = []
    for v in range(1 << len(qubits)):
        s = dict(base)
        for i, q in enumerate(qubits):
            s[q] = (v >> (len(qubits) - 1 - i)) & 1
        out.append("".join(str(s[q]) for q in closed))
    return out


def test_unpinned_network_reproduces_repin(workloads):
    from paper_2103_03074_b200.batched import batched_network

    w = workloads("m12")
    closed = sorted(w.tn.fixed_output_bits)
    qs = [closed[1], closed[4], closed[7]]
    s1s = _s1_list(w.tn, qs)
    tnb, order, q_ix, base, norm = batched_network(w.tn, s1s)
    assert order == qs and len(q_ix) == 3
    for s in norm:
        ref = w.tn.repin(s)
        for nid, node in tnb.nodes.items():
            data = np.asarray(node.data)
            ids = list(node.indices)
            for q, ix in zip(order, q_ix):
                if ix in ids:
                    ax = ids.index(ix)
                    data = np.take(data, s[q], axis=ax)
                    del ids[ax]
            assert ids == list(ref.nodes[nid].indices)
            assert np.array_equal(data, np.asarray(ref.nodes[nid].data))


@pytest.mark.gpu
@pytest.mark.parametrize("name,nq,precision", [("s8", 2, "double"), ("s8", 3, "single"),
                                               ("m12", 2, "single"), ("c2", 3, "single")])
def test_batched_head_vectors_match_per_s1(gpu, workloads, name, nq, precision):
    import paper_2103_03074_b200 as tnb
    from paper_2103_03074_b200.batched import compute_head_vectors_batched

    w = workloads(name)
    closed = sorted(w.tn.fixed_output_bits)
    s1s = _s1_list(w.tn, closed[:nq])
    rng_ = (0, 2)
    hvs = compute_head_vectors_batched(w.tn, w.tree, w.sliced, s1s, slice_range=rng_,
                                       precision=precision)
    # single: both sides carry fp32 rounding of their own (c2 is 3.6e-5 from
    # fp64 even on the pure fp32 SIMT path), so the north-star tolerance
    tol = 1e-10 if precision == "double" else 1e-4
    assert len(hvs) == len(s1s)
    for s, hv in zip(s1s, hvs):
        ref = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s, slice_range=rng_, precision=precision)
        assert hv.provenance == ref.provenance and hv.s1 == ref.s1
        assert rel_l2(hv.data, ref.data) < tol
        ta = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision=precision)
        tr = tnb.tail_amplitudes_unchecked(w.tn, w.tree, ref, precision=precision)
        assert rel_l2(ta.amplitudes, tr.amplitudes) < tol
