"""Host-side logic and the C-ABI surface (CPU only)."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import ROOT, import_reference


def _header_symbols():
    with open(os.path.join(ROOT, "include", "tnb.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(tnb_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    from paper_2103_03074_b200 import _lib

    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.EXPORTS, s
    assert lib.tnb_abi_version() == 2


def test_no_device_fails_loudly_not_silently():
    from paper_2103_03074_b200 import _lib

    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError):
        _lib.require_device()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2103_03074_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_provenance_matches_reference(workloads):
    tncut = import_reference()
    from tncut import engine as teng
    from tncut import ordering as tord
    from tncut.circuit import parse_circuit
    from tncut.network import build_network

    from paper_2103_03074_b200.provenance import provenance_hash

    for name in ("c1", "s8", "c4"):
        w = workloads(name)
        with open(os.path.join(ROOT, "tests", "golden", name, "circuit.qsim")) as fh:
            c = parse_circuit(fh.read(), "qsim_text")
        opens = w.doc["open_qubits"]
        tn = build_network(c, set(opens), {q: 0 for q in c.layout.ids if q not in set(opens)})
        tree = tord.doc_to_tree(w.doc)
        s1 = dict(tn.fixed_output_bits)
        for prec, mode in (("double", "fixed"), ("single", "free")):
            ref = teng.provenance_hash(tn, tree, s1, prec, mode, w.sliced)
            ours_ref_objs = provenance_hash(tn, tree, s1, prec, mode, w.sliced)
            ours_frozen = provenance_hash(w.tn, w.tree, s1, prec, mode, w.sliced)
            assert ref == ours_ref_objs == ours_frozen


def test_frozen_repin_matches_reference_build(workloads):
    import_reference()
    from tncut.circuit import parse_circuit
    from tncut.network import build_network

    w = workloads("c1")
    with open(os.path.join(ROOT, "tests", "golden", "c1", "circuit.qsim")) as fh:
        c = parse_circuit(fh.read(), "qsim_text")
    opens = w.doc["open_qubits"]
    rng = np.random.default_rng(0)
    for _ in range(5):
        bits = {q: int(rng.integers(2)) for q in w.tn.fixed_output_bits}
        ref = build_network(c, set(opens), bits)
        ours = w.tn.repin(bits)
        assert sorted(ref.nodes) == sorted(ours.nodes)
        for nid in ref.nodes:
            assert ref.nodes[nid].indices == ours.nodes[nid].indices
            assert np.array_equal(ref.nodes[nid].data, ours.nodes[nid].data)


def test_tail_order_is_valid_and_no_worse_than_reference_greedy(workloads):
    """The head-absorbed tail's order (native planner, treeopt.order_network)
    contracts every tail leaf + the head leaf exactly once, keeps the open
    legs, and is no slower under the B200 time model than the reference's
    greedy order (restated in the oracle, ordering.py:256-285)."""
    from oracle import engine_np as O
    from paper_2103_03074_b200.planner import split
    from paper_2103_03074_b200.treeopt import order_network

    def model(sets, steps):
        s = {k: frozenset(v) for k, v in sets.items()}
        t = 0.0
        for l, r, o in steps:
            a, b = s.pop(l), s.pop(r)
            s[o] = a ^ b
            t += max(8 * 2 ** len(a | b) / 4.1e14,
                     8 * (2 ** len(a) + 2 ** len(b) + 2 ** len(s[o])) / 4e12) + 5e-6
        return t, s

    for name in ("c1", "s8", "c2", "c4"):
        w = workloads(name)
        _, _, tail, _, cut = split(w.tn, w.tree)
        hid = max(w.tn.nodes) + 1
        sets = {n: w.tn.nodes[n].indices for n in tail}
        sets[hid] = list(cut)
        ours = order_network(sets, hid + 1)
        assert [o for _, _, o in ours] == list(range(hid + 1, hid + len(sets)))
        t_ours, rest = model(sets, ours)
        assert len(rest) == 1
        assert set(next(iter(rest.values()))) == set(w.tn.open_output_indices.values())
        t_ref, _ = model(sets, O.greedy_steps(sets, hid + 1))
        assert t_ours <= t_ref * (1 + 1e-9), name


def test_split_and_stats_analytic(workloads):
    """Analytic multiplication counts == the oracle's executed counts."""
    from oracle import engine_np as O
    from paper_2103_03074_b200.planner import split, step_mults

    w = workloads("s8")
    h, hs, t, ts, cut = split(w.tn, w.tree)
    oh, ohs, ot, ots, ocut = O.split(w.tn, w.tree)
    assert (h, t, cut) == (oh, ot, ocut)
    assert [(s.lhs, s.rhs, s.out) for s in hs] == [(s.lhs, s.rhs, s.out) for s in ohs]
    st = O.Stats()
    O.head_vector(w.tn, w.tree, w.sliced, (0, 1), "single", stats=st)
    mults, _ = step_mults({n: w.tn.nodes[n].indices for n in h}, hs, frozenset(w.sliced))
    assert mults == st.multiplications == w.tc_per_slice


def test_tree_doc_roundtrip(workloads):
    from paper_2103_03074_b200.provenance import dumps_order
    from paper_2103_03074_b200.types import tree_to_doc

    w = workloads("c4")
    doc = tree_to_doc(w.tree, circuit_sha256=w.doc["circuit_sha256"],
                      open_qubits=w.doc["open_qubits"], slices=w.doc["slices"],
                      subtask=w.doc["subtask"])
    with open(os.path.join(ROOT, "tests", "golden", "c4", "order.json")) as fh:
        assert dumps_order(doc) == fh.read()


def test_thread_devices_round_robin(monkeypatch):
    """set_thread_devices: each calling thread gets the next device (the
    reference CLI's --threads workers spread over the GPUs); an explicit
    device argument always wins; off -> the process default."""
    import threading

    from paper_2103_03074_b200 import _lib, engine as E

    monkeypatch.setattr(_lib, "device_count", lambda: 4)
    monkeypatch.setattr(E, "_thread_counter", [0])
    E.set_thread_devices(True)
    try:
        seen = []

        def work():
            d1 = E._resolve_device(None)
            d2 = E._resolve_device(None)  # sticky per thread
            seen.append((d1, d2, E._resolve_device(7)))

        th = [threading.Thread(target=work) for _ in range(6)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert all(a == b and c == 7 for a, b, c in seen)
        assert sorted(a for a, _, _ in seen) == [0, 0, 1, 1, 2, 3]
    finally:
        E.set_thread_devices(False)
    assert E._resolve_device(None) == E._default_device
