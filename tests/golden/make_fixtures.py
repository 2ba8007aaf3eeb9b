"""Freeze the parity fixtures from the reference package (run HERE only).

This script imports the reference ``tncut`` package from
``/root/reference/pkg/src`` (read-only) and writes, per config, the
frozen inputs the B200 executor and the oracle consume on machines where
the reference does not exist (the GPU box):

* ``network.json`` -- the fused tensor network (``network.py:113-218``)
  with the closed-qubit nodes also stored *unpinned* so that ``repin``
  (``network.py:65-77``) can be replayed without the circuit builder;
* ``order.json``   -- the sliced order document exactly as ``tncut slice``
  writes it (``cli.py:270-298`` / ``ordering.py:670-722``);
* ``circuit.qsim`` -- the circuit text (``circuit.py:435-449``).

Stage ``goldens`` then drives the reference engine
(``engine.py:242-378``) and the state-vector oracle
(``statevector.py:27-42``) to produce ``golden_*.npz`` known-answer
vectors.  Planner settings follow SURVEY.md section 8 (config key).

Usage:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fixtures.py plans [names]
        PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fixtures.py goldens [names]
"""

from __future__ import annotations

import base64
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from tncut import circuit as tcircuit  # noqa: E402
from tncut import engine as tengine  # noqa: E402
from tncut import ordering as tordering  # noqa: E402
from tncut import sycamore as tsyc  # noqa: E402
from tncut.network import build_network  # noqa: E402
from tncut.slicing import select_slices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# Circuits

def grid_circuit(rows: int, cols: int, cycles: int, seed: int = 0,
                 sequence: str = "ABCDCDAB") -> tcircuit.Circuit:
    """3x4-grid analogue of ``sycamore_circuit`` (sycamore.py:87-136).

    Coordinates (r, c), numbered row-major; couplers are grid-adjacent
    pairs; pattern from ``coupler_pattern`` (sycamore.py:60-67); the
    single-qubit layers and per-coupler angles follow sycamore_circuit.
    """
    coords = [(r, c) for r in range(rows) for c in range(cols)]
    index = {rc: i for i, rc in enumerate(coords)}
    pairs = []
    for (r, c), i in index.items():
        for nb in ((r + 1, c), (r, c + 1)):
            if nb in index:
                pairs.append((i, index[nb]))
    pairs.sort()
    pats = {"A": [], "B": [], "C": [], "D": []}
    for i, j in pairs:
        pats[tsyc.coupler_pattern(coords[i], coords[j])].append((i, j))
    n = len(coords)
    rng = np.random.default_rng(seed)
    angles = {
        pair: (math.pi / 2 + rng.uniform(-0.1, 0.1), math.pi / 6 + rng.uniform(-0.1, 0.1))
        for pair in pairs
    }
    gates = (tcircuit.GateKind.SQRT_X, tcircuit.GateKind.SQRT_Y, tcircuit.GateKind.SQRT_W)
    last = [-1] * n
    moments = []

    def single_layer():
        layer = []
        for q in range(n):
            choices = [k for k in range(3) if k != last[q]]
            pick = choices[rng.integers(len(choices))]
            last[q] = pick
            layer.append(tcircuit.GateSpec(gates[pick], (q,)))
        return layer

    for cycle in range(cycles):
        moments.append(single_layer())
        pat = sequence[cycle % len(sequence)]
        moments.append([tcircuit.GateSpec(tcircuit.GateKind.FSIM, p, angles[p])
                        for p in pats[pat]])
    moments.append(single_layer())
    return tcircuit.Circuit(layout=tcircuit.QubitLayout.linear(n), moments=moments,
                            metadata={"device": f"grid{rows}x{cols}", "seed": seed,
                                      "cycles": cycles})


# name -> (circuit factory, open qubits, planner seed, restarts, target space)
CONFIGS = {
    # C1: SURVEY 8(d) -- 3x4 grid, m=8, open {0,1,4,5}, restarts 4, t=2^8
    "c1": (lambda: grid_circuit(3, 4, 8, seed=0), [0, 1, 4, 5], 0, 4, 8),
    # small Sycamore-53 slice for fast CPU+GPU parity (SIMT-size steps)
    "s8": (lambda: tsyc.sycamore_circuit(8, seed=0),
           sorted(tsyc.OPEN_QUBITS_M20)[:12], 0, 4, 18),
    # m=12, 21 open, target 2^24 (3.85 s/slice single on 8 cores)
    "m12": (lambda: tsyc.sycamore_circuit(12, seed=0),
            sorted(tsyc.OPEN_QUBITS_M20)[:21], 0, 8, 24),
    # C2: m=12, n2=10, seed 2 / restarts 8 / t=2^28
    "c2": (lambda: tsyc.sycamore_circuit(12, seed=0),
           sorted(tsyc.OPEN_QUBITS_M20)[:10], 2, 8, 28),
    # C3: m=14, n2=16, seed 0 / restarts 16 / t=2^30
    "c3": (lambda: tsyc.sycamore_circuit(14, seed=0),
           sorted(tsyc.OPEN_QUBITS_M20)[:16], 0, 16, 30),
    # C4: m=20, n2=20, seed 0 / restarts 16 / t=2^30  (bench workload)
    "c4": (lambda: tsyc.sycamore_circuit(20, seed=0),
           sorted(tsyc.OPEN_QUBITS_M20)[:20], 0, 16, 30),
    # C5: the C4 tree re-sliced at other space targets (sliced-edge sweep,
    # SURVEY 8(d)): t=26/28/32 -> n_e 63/58/48
    "c5_26": (lambda: tsyc.sycamore_circuit(20, seed=0),
              sorted(tsyc.OPEN_QUBITS_M20)[:20], 0, 16, 26),
    "c5_28": (lambda: tsyc.sycamore_circuit(20, seed=0),
              sorted(tsyc.OPEN_QUBITS_M20)[:20], 0, 16, 28),
    "c5_32": (lambda: tsyc.sycamore_circuit(20, seed=0),
              sorted(tsyc.OPEN_QUBITS_M20)[:20], 0, 16, 32),
    # C5 batch-size axis: 2^21 correlated bitstrings (all OPEN_QUBITS_M20), t=30
    "c5_n21": (lambda: tsyc.sycamore_circuit(20, seed=0),
               sorted(tsyc.OPEN_QUBITS_M20)[:21], 0, 16, 30),
}


def _b64(a: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(a, dtype=np.complex128).tobytes()).decode()


def network_doc(c, tn) -> dict:
    """Network + unpinned closed-output nodes (for repin without a builder)."""
    tn_open = build_network(c, set(c.layout.ids), {})
    fixed_node = tn.metadata["fixed_output_node"]
    unpinned = {}
    for q, nid in fixed_node.items():
        node_open = tn_open.nodes[nid]
        ent = unpinned.setdefault(nid, {"indices": list(node_open.indices),
                                        "shape": list(node_open.data.shape),
                                        "data_b64": _b64(node_open.data),
                                        "qubits": {}})
        ent["qubits"][str(q)] = tn_open.open_output_indices[q]
    # self-check: np.take on the unpinned node reproduces the pinned one
    for nid, ent in unpinned.items():
        data = tn_open.nodes[nid].data
        ids = list(ent["indices"])
        for q, ix in ent["qubits"].items():
            ax = ids.index(ix)
            data = np.take(data, tn.fixed_output_bits[int(q)], axis=ax)
            del ids[ax]
        assert ids == tn.nodes[nid].indices, (nid, ids, tn.nodes[nid].indices)
        assert np.array_equal(data, tn.nodes[nid].data)
    return {
        "schema": "tnb-network/1",
        "nodes": [
            {"id": n.id, "indices": list(n.indices), "shape": list(n.data.shape),
             "data_b64": _b64(n.data)}
            for n in tn.nodes.values()
        ],
        "open_output_indices": {str(k): v for k, v in tn.open_output_indices.items()},
        "fixed_output_bits": {str(k): v for k, v in tn.fixed_output_bits.items()},
        "fixed_output_node": {str(k): v for k, v in fixed_node.items()},
        "unpinned": {str(k): v for k, v in unpinned.items()},
        "circuit_sha256": c.sha256(),
        "layout_ids": list(c.layout.ids),
    }


def make_plan(name: str) -> None:
    factory, opens, seed, restarts, target = CONFIGS[name]
    out = os.path.join(HERE, name)
    os.makedirs(out, exist_ok=True)
    c = factory()
    t0 = time.time()
    fixed = {q: 0 for q in c.layout.ids if q not in set(opens)}
    tn = build_network(c, set(opens), fixed)
    cons = tordering.PartitionConstraints(rng_seed=seed, restarts=restarts)
    tree = tordering.hierarchical_partition(tn, cons)
    plan, tree = select_slices(tn, tree, target, reconfigure=True)
    n2 = len(opens)
    subtask = {
        "count": plan.subtask_count,
        "n_e": len(plan.sliced_indices),
        "tc": plan.per_subtask.tc,
        "sc_log2": plan.per_subtask.sc_log2,
        "overhead": plan.overhead,
        "target_space": target,
        "t_head": plan.subtask_count * plan.per_subtask.tc,
    }
    if plan.tail_per_assignment is not None:
        subtask["tail_tc"] = plan.tail_per_assignment.tc
        subtask["tail_sc_log2"] = plan.tail_per_assignment.sc_log2
        subtask["t_tail"] = (1 << n2) * plan.tail_per_assignment.tc
        subtask["t_total"] = subtask["t_head"] + subtask["t_tail"]
    doc = tordering.tree_to_doc(tree, circuit_sha256=c.sha256(), open_qubits=opens,
                                slices=plan.sliced_indices, subtask=subtask)
    with open(os.path.join(out, "order.json"), "w") as fh:
        fh.write(tordering.dumps_order(doc))
    with open(os.path.join(out, "network.json"), "w") as fh:
        json.dump(network_doc(c, tn), fh, sort_keys=True)
    with open(os.path.join(out, "circuit.qsim"), "w") as fh:
        fh.write(tcircuit.to_qsim_text(c))
    head, tail = tree.head_tail_leaves()
    cut = tordering.cut_indices(tn, set(head), set(tail))
    print(f"[{name}] plan in {time.time() - t0:.1f}s: n_e={len(plan.sliced_indices)} "
          f"n_c={len(cut)} tc=2^{math.log2(plan.per_subtask.tc):.2f} "
          f"head/tail={len(head)}/{len(tail)} steps={len(tree.head_steps())}", flush=True)


if __name__ == "__main__":
    stage = sys.argv[1]
    names = sys.argv[2:] or list(CONFIGS)
    if stage == "plans":
        for n in names:
            make_plan(n)
    elif stage == "goldens":
        from make_goldens import make_golden  # noqa: E402
        for n in names:
            make_golden(n)
    else:
        raise SystemExit(f"unknown stage {stage}")
