"""Known-answer vectors from the reference engine (run HERE only).

Drives the unmodified reference ``tncut`` engine on the frozen fixtures
written by ``make_fixtures.py`` and stores the results as ``golden.npz``
per config.  Everything here is produced by reference code paths:

* head partials: ``compute_head_vector`` (engine.py:242-310);
* blocked tail: ``compute_tail_amplitudes`` (engine.py:313-378), fed a
  partial with ``slice_range`` replaced by the full range;
* head-absorbed tail (configs whose blocked tail is infeasible on CPU):
  the tail leaves plus one node carrying the head vector, ordered by the
  reference ``greedy_order`` (ordering.py:238-285) and contracted by the
  reference ``contract_tree`` (engine.py:147-165);
* C1 amplitudes additionally from the state-vector oracle
  (statevector.py:27-42 via tests/conftest.py:13-36 semantics).

Large vectors are stored subsampled (every ``stride``-th entry) plus
their exact squared L2 norm so fixtures stay small.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from tncut import engine as tengine  # noqa: E402
from tncut import ordering as tordering  # noqa: E402
from tncut.circuit import parse_circuit  # noqa: E402
from tncut.network import TensorNetwork, TensorNode, build_network  # noqa: E402
from tncut.statevector import simulate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    d = os.path.join(HERE, name)
    with open(os.path.join(d, "circuit.qsim")) as fh:
        c = parse_circuit(fh.read(), "qsim_text")
    with open(os.path.join(d, "order.json")) as fh:
        doc = json.load(fh)
    tree = tordering.doc_to_tree(doc)
    opens = doc["open_qubits"]
    fixed = {q: 0 for q in c.layout.ids if q not in set(opens)}
    tn = build_network(c, set(opens), fixed)
    assert c.sha256() == doc["circuit_sha256"]
    return c, tn, tree, doc


def absorbed_tail(tn, tree, head_data, cut, dtype):
    """Reference-built head-absorbed tail: greedy_order + contract_tree."""
    _, tail_leaves = tree.head_tail_leaves()
    nodes = {nid: tn.nodes[nid] for nid in sorted(tail_leaves)}
    hid = max(tn.nodes) + 1
    nodes[hid] = TensorNode(id=hid, indices=list(cut),
                            data=np.asarray(head_data, dtype=np.complex128).reshape((2,) * len(cut)),
                            origin="head")
    sub = TensorNetwork(nodes=nodes, index_endpoints={},
                        open_output_indices=dict(tn.open_output_indices),
                        fixed_output_bits={}, circuit=None)
    sub.index_endpoints = sub.recompute_endpoints()
    gtree = tordering.greedy_order(sub)
    res = tengine.contract_tree(sub, gtree, {}, dtype=dtype)
    # contract_tree sorts open axes by index id; reorder to open qubits ascending
    opens = sorted(tn.open_output_indices)
    ids = sorted(tn.open_output_indices[q] for q in opens)
    order = [ids.index(tn.open_output_indices[q]) for q in opens]
    return np.transpose(res, order).reshape(-1)


def sub(x, stride):
    x = np.asarray(x)
    return x[::stride].copy(), float(np.vdot(x, x).real)


def make_golden(name):
    c, tn, tree, doc = load(name)
    sliced = doc["slices"]
    n_e = len(sliced)
    out = {}
    t0 = time.time()
    head_leaves, _ = tree.head_tail_leaves()
    _, _, _, _, cut = tengine._split(tn, tree)
    if name == "c1":
        opens = doc["open_qubits"]
        closed = [q for q in c.layout.ids if q not in set(opens)]
        sv = simulate(c).data
        amps_sv, amps_eng = [], []
        for s1v in range(1 << len(closed)):
            s1 = "".join(str((s1v >> (len(closed) - 1 - i)) & 1) for i in range(len(closed)))
            hv = tengine.compute_head_vector(tn, tree, sliced, s1, precision="double")
            tab = tengine.compute_tail_amplitudes(tn, tree, hv, space_cap=8, precision="double")
            amps_eng.append(tab.amplitudes)
            row = np.zeros(1 << len(opens), dtype=complex)
            s1d = {q: int(b) for q, b in zip(closed, s1)}
            for mask in range(1 << len(opens)):
                index = 0
                for q in sorted(c.layout.ids):
                    bit = s1d[q] if q in s1d else (mask >> (len(opens) - 1 - opens.index(q))) & 1
                    index = (index << 1) | bit
                row[mask] = sv[index]
            amps_sv.append(row)
        out["amps_engine"] = np.array(amps_eng)
        out["amps_statevector"] = np.array(amps_sv)
        st = tengine.EngineStats()
        hv = tengine.compute_head_vector(tn, tree, sliced, None, precision="double", stats=st)
        out["head_full_double"] = hv.data
        out["head_stats"] = np.array([st.multiplications, st.head_contractions, 0, st.steps_executed])
        st2 = tengine.EngineStats()
        tab = tengine.compute_tail_amplitudes(tn, tree, hv, space_cap=8, precision="double", stats=st2)
        out["tail_stats"] = np.array([st2.multiplications, 0, st2.tail_contractions, st2.steps_executed])
        out["tail_stats_cap6"] = None
        st3 = tengine.EngineStats()
        tengine.compute_tail_amplitudes(tn, tree, hv, space_cap=6, precision="double", stats=st3)
        out["tail_stats_cap6"] = np.array([st3.multiplications, 0, st3.tail_contractions, st3.steps_executed])
        out["provenance"] = np.array(hv.provenance)
        for a, b in [(0, 8), (8, 16), (0, 4), (4, 8), (3, 11)]:
            for mode in ("fixed", "free"):
                p = tengine.compute_head_vector(tn, tree, sliced, None, slice_range=(a, b),
                                                precision="double", mode=mode)
                out[f"head_{mode}_{a}_{b}"] = p.data
        hs = tengine.compute_head_vector(tn, tree, sliced, None, precision="single")
        out["head_full_single"] = hs.data
        out["amps_single"] = tengine.compute_tail_amplitudes(tn, tree, hs, precision="single").amplitudes
        # whole-tree contraction with a fixed assignment (contract_tree, engine.py:147-165)
        asg = {ix: (5 >> (n_e - 1 - p)) & 1 for p, ix in enumerate(sliced)}
        out["contract_tree_mask5"] = tengine.contract_tree(tn, tree, asg)
    elif name == "c1_opt":
        # co-optimised plan (treeopt): the full slice sum is plan-independent,
        # so it must equal c1's head vector and amplitudes
        hv = tengine.compute_head_vector(tn, tree, sliced, None, precision="double")
        out["head_full_double"] = hv.data
        out["amps_double"] = tengine.compute_tail_amplitudes(tn, tree, hv, space_cap=8,
                                                             precision="double").amplitudes
        for a, b in [(0, 1), (1, 4)]:
            out[f"head_fixed_{a}_{b}"] = tengine.compute_head_vector(
                tn, tree, sliced, None, slice_range=(a, b), precision="double").data
    else:
        ranges = {"s8": [(0, 4), (0, 1), (4, 8)], "s8_opt": [(0, 4), (0, 1)], "c4_opt": [(0, 1)], "c4_opt_b200": [(0, 1)], "c4_opt31_b200": [(0, 1)], "c2_opt_b200": [(0, 1)], "c3_opt_b200": [(0, 1)], "m12": [(0, 1)], "c2": [(0, 1)],
                  "c3": [(0, 1)], "c4": [(0, 1)], "c5_26": [(0, 2)], "c5_28": [(0, 1)],
                  "c5_n21": [(0, 1)]}[name]
        stride = {"s8_opt": 32, "c4_opt": 64, "c4_opt_b200": 64, "c4_opt31_b200": 64, "c2_opt_b200": 1, "c3_opt_b200": 4, "s8": 32, "m12": 64, "c2": 1, "c3": 4, "c4": 64, "c5_26": 64, "c5_28": 64,
                  "c5_n21": 64}[name]
        for (a, b) in ranges:
            st = tengine.EngineStats()
            t1 = time.time()
            p = tengine.compute_head_vector(tn, tree, sliced, None, slice_range=(a, b),
                                            precision="single", mode="fixed", stats=st)
            dt = time.time() - t1
            print(f"[{name}] head [{a},{b}) single: {dt:.1f}s", flush=True)
            out[f"head_single_{a}_{b}_sub"], out[f"head_single_{a}_{b}_norm2"] = sub(p.data, stride)
            out[f"head_single_{a}_{b}_stats"] = np.array([st.multiplications, st.head_contractions,
                                                          0, st.steps_executed])
            out[f"head_single_{a}_{b}_cpu_s"] = np.array(dt)
            if name in ("s8", "m12", "s8_opt"):
                pd = tengine.compute_head_vector(tn, tree, sliced, None, slice_range=(a, b),
                                                 precision="double", mode="fixed")
                out[f"head_double_{a}_{b}_sub"], out[f"head_double_{a}_{b}_norm2"] = sub(pd.data, stride)
            if (a, b) == ranges[0]:
                full = dataclasses.replace(p, slice_range=(0, 1 << n_e))
                amp_stride = {"s8_opt": 1, "c4_opt": 16, "c4_opt_b200": 16, "c4_opt31_b200": 16, "c2_opt_b200": 1, "c3_opt_b200": 16, "s8": 1, "m12": 256, "c2": 1, "c3": 16, "c4": 16, "c5_26": 16,
                              "c5_28": 16, "c5_n21": 32}[name]
                if name in ("s8", "c2", "s8_opt"):
                    t1 = time.time()
                    tab = tengine.compute_tail_amplitudes(tn, tree, full, space_cap=30,
                                                          precision="single")
                    amps = tab.amplitudes
                    print(f"[{name}] blocked tail: {time.time() - t1:.1f}s", flush=True)
                else:
                    t1 = time.time()
                    amps = absorbed_tail(tn, tree, p.data, sorted(cut), np.complex128)
                    print(f"[{name}] absorbed tail: {time.time() - t1:.1f}s", flush=True)
                out["amps_sub"], out["amps_norm2"] = sub(amps, amp_stride)
                out["amps_stride"] = np.array(amp_stride)
                out["amps_probsum"] = np.array(float(np.sum(np.abs(amps) ** 2)))
                if name == "s8":
                    # both tails agree: pins the head-absorbed formulation itself
                    out["amps_absorbed"] = absorbed_tail(tn, tree, p.data, sorted(cut), np.complex128)
        out["stride"] = np.array(stride)
    out = {k: v for k, v in out.items() if v is not None}
    np.savez_compressed(os.path.join(HERE, name, "golden.npz"), **out)
    print(f"[{name}] goldens in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        make_golden(n)
