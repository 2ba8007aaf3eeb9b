"""TNCUTHV1 / TSV interop with the reference writers (CPU)."""

from __future__ import annotations

import dataclasses
import os

import numpy as np

from conftest import golden, import_reference


def _head(w, data, rng_, mode="fixed"):
    from paper_2103_03074_b200.provenance import provenance_hash
    from paper_2103_03074_b200.types import HeadVector

    s1 = dict(w.tn.fixed_output_bits)
    return HeadVector(s1=s1, data=data, provenance=provenance_hash(w.tn, w.tree, s1, "double", mode,
                                                                   w.sliced),
                      cut_order=sorted(__import__("paper_2103_03074_b200.planner", fromlist=["x"])
                                       .split(w.tn, w.tree)[4]),
                      n_e=w.n_e, slice_range=rng_, mode=mode, sliced_indices=tuple(w.sliced))


def test_head_vector_roundtrip_and_reference_bytes(tmp_path, workloads):
    from paper_2103_03074_b200 import io

    w = workloads("c1")
    g = golden("c1")
    hv = _head(w, g["head_fixed_0_8"], (0, 8))
    p = tmp_path / "ours.hv"
    io.write_head_vector(p, hv)
    back = io.read_head_vector(p)
    assert np.array_equal(back.data, hv.data) and back.slice_range == (0, 8)
    assert back.provenance == hv.provenance and back.cut_order == hv.cut_order
    tncut = import_reference()
    from tncut import engine as teng

    q = tmp_path / "ref.hv"
    teng.write_head_vector(q, hv)
    assert p.read_bytes() == q.read_bytes()
    ref_back = teng.read_head_vector(p)
    assert np.array_equal(ref_back.data, hv.data)


def test_file_partials_reduce_like_reference(tmp_path, workloads):
    """run --slices A..B + reduce through files (cli.py:358-365, 417-441)."""
    from oracle import engine_np as O
    from paper_2103_03074_b200 import io

    w = workloads("c1")
    g = golden("c1")
    paths = []
    for a in (0, 8):
        hv = _head(w, g[f"head_fixed_{a}_{a + 8}"], (a, a + 8))
        paths.append(tmp_path / f"p{a}.hv")
        io.write_head_vector(paths[-1], hv)
    parts = [io.read_head_vector(p) for p in paths]
    tncut = import_reference()
    from tncut import engine as teng

    red = teng.reduce_partials(parts)
    assert np.array_equal(red.data, g["head_full_double"])
    assert np.array_equal(O.combine_partials([(p.slice_range, p.data) for p in parts]),
                          g["head_full_double"])


def test_amplitude_tsv_byte_identical(tmp_path, workloads):
    from paper_2103_03074_b200 import io

    tncut = import_reference()
    from tncut import engine as teng

    w = workloads("c1")
    g = golden("c1")
    for amps in (g["amps_engine"][0], g["amps_single"]):
        tab = teng.AmplitudeTable(s1=dict(w.tn.fixed_output_bits),
                                  open_qubits=sorted(w.tn.open_output_indices), amplitudes=amps,
                                  layout_ids=list(range(12)), circuit_sha256="c" * 64,
                                  order_sha256="o" * 64, precision="double", mode="fixed")
        a, b = tmp_path / "ours.tsv", tmp_path / "ref.tsv"
        io.write_amplitude_tsv(a, tab)
        teng.write_amplitude_tsv(b, tab)
        assert a.read_bytes() == b.read_bytes()
        assert list(io.bitstrings(tab)) == [tab.bitstring(m).encode() for m in range(len(amps))]


def test_amplitude_tsv_byte_identical_at_scale(tmp_path):
    """2^16 rows of random c64 / c128 amplitudes spanning 2^-60..2^7 plus
    zeros, -0, subnormals, +-inf and NaN: the libtnbio writer equals the
    reference's per-row Python writer byte for byte (probability column:
    numpy scalar abs ** 2 = libm hypotf/powf, not h*h)."""
    from paper_2103_03074_b200 import io

    import_reference()
    from tncut import engine as teng

    rng = np.random.default_rng(11)
    n2 = 16
    for dt in (np.complex64, np.complex128):
        a = (rng.standard_normal(1 << n2) + 1j * rng.standard_normal(1 << n2)) * \
            np.exp(rng.uniform(-42, 5, 1 << n2))
        a = a.astype(dt)
        a[:8] = [0, -0.0, 1e-45, np.inf, -np.inf, complex(np.nan, 1), complex(-np.nan, -0.0), 3e38]
        s1 = {q: q % 2 for q in range(n2, 53)}
        tab = teng.AmplitudeTable(s1=s1, open_qubits=list(range(n2)), amplitudes=a,
                                  layout_ids=list(range(53)), circuit_sha256="c" * 64,
                                  order_sha256="o" * 64, precision="single", mode="fixed")
        ours, ref = tmp_path / "ours.tsv", tmp_path / "ref.tsv"
        io.write_amplitude_tsv(ours, tab)
        with np.errstate(all="ignore"):
            teng.write_amplitude_tsv(ref, tab)
        assert ours.read_bytes() == ref.read_bytes(), dt
