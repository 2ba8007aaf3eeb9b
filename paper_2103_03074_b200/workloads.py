"""Frozen workloads: networks + sliced orders produced by the reference.

The reference planner (circuit -> network -> order -> slices) is host-side
and out of scope; its outputs for the BASELINE configs are frozen under
``tests/golden/<name>/`` by ``tests/golden/make_fixtures.py``.  This module
rebuilds duck-typed ``TensorNetwork`` / ``ContractionTree`` objects from
them so the executor runs where ``tncut`` is not installed (the GPU box).

``FrozenNetwork.repin`` replays ``TensorNetwork.repin``
(network.py:65-77): the closed-output nodes are stored unpinned and the
basis projection of ``pin_basis`` (network.py:103-105, np.take + drop the
axis) is re-applied for the new bits.
"""

from __future__ import annotations

import base64
import json
import os
from dataclasses import dataclass, field

import numpy as np

from .types import doc_to_tree

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "tests", "golden")


def _decode(b64: str, shape) -> np.ndarray:
    return np.frombuffer(base64.b64decode(b64), dtype=np.complex128).reshape(shape).copy()


@dataclass
class FrozenNode:
    id: int
    indices: list
    data: np.ndarray
    origin: str = "frozen"

    @property
    def rank(self) -> int:
        return len(self.indices)


@dataclass
class _Layout:
    ids: tuple


class FrozenCircuit:
    """Just what the engine reads from ``tn.circuit``: sha256 and layout."""

    def __init__(self, sha: str, layout_ids):
        self._sha = sha
        self.layout = _Layout(tuple(layout_ids))

    def sha256(self) -> str:
        return self._sha


@dataclass
class FrozenNetwork:
    nodes: dict
    index_endpoints: dict
    open_output_indices: dict
    fixed_output_bits: dict
    circuit: FrozenCircuit | None = None
    metadata: dict = field(default_factory=dict)
    _unpinned: dict = field(default_factory=dict, repr=False)

    @property
    def n_open(self) -> int:
        return len(self.open_output_indices)

    def recompute_endpoints(self) -> dict:
        eps: dict = {}
        for node in self.nodes.values():
            for ix in node.indices:
                eps.setdefault(ix, []).append(node.id)
        return {ix: tuple(v) for ix, v in eps.items()}

    def repin(self, fixed_bits: dict) -> "FrozenNetwork":
        if set(fixed_bits) != set(self.fixed_output_bits):
            raise ValueError("fixed-bit qubit set differs from the network's")
        if dict(fixed_bits) == self.fixed_output_bits:
            return self
        nodes = dict(self.nodes)
        for nid, ent in self._unpinned.items():
            data = ent["data"]
            ids = list(ent["indices"])
            for q, ix in ent["qubits"].items():
                ax = ids.index(ix)
                data = np.take(data, int(fixed_bits[q]), axis=ax)
                del ids[ax]
            nodes[nid] = FrozenNode(id=nid, indices=ids, data=np.ascontiguousarray(data))
        tn = FrozenNetwork(nodes=nodes, index_endpoints=self.index_endpoints,
                           open_output_indices=dict(self.open_output_indices),
                           fixed_output_bits={q: int(b) for q, b in fixed_bits.items()},
                           circuit=self.circuit, metadata=dict(self.metadata),
                           _unpinned=self._unpinned)
        return tn


def load_network(path: str) -> FrozenNetwork:
    with open(path) as fh:
        doc = json.load(fh)
    nodes = {}
    for nd in doc["nodes"]:
        nodes[nd["id"]] = FrozenNode(id=nd["id"], indices=list(nd["indices"]),
                                     data=_decode(nd["data_b64"], nd["shape"]))
    unpinned = {}
    for nid, ent in doc.get("unpinned", {}).items():
        unpinned[int(nid)] = {
            "indices": list(ent["indices"]),
            "data": _decode(ent["data_b64"], ent["shape"]),
            "qubits": {int(q): ix for q, ix in ent["qubits"].items()},
        }
    tn = FrozenNetwork(
        nodes=nodes,
        index_endpoints={},
        open_output_indices={int(k): v for k, v in doc["open_output_indices"].items()},
        fixed_output_bits={int(k): v for k, v in doc["fixed_output_bits"].items()},
        circuit=FrozenCircuit(doc["circuit_sha256"], doc["layout_ids"]),
        metadata={"fixed_output_node": {int(k): v for k, v in doc["fixed_output_node"].items()},
                  "open_qubits": sorted(int(k) for k in doc["open_output_indices"])},
        _unpinned=unpinned,
    )
    tn.index_endpoints = tn.recompute_endpoints()
    return tn


@dataclass
class Workload:
    name: str
    tn: FrozenNetwork
    tree: object
    doc: dict

    @property
    def sliced(self) -> list:
        return list(self.doc.get("slices", []))

    @property
    def n_e(self) -> int:
        return len(self.sliced)

    @property
    def tc_per_slice(self) -> int:
        return int(self.doc["subtask"]["tc"])

    @property
    def target_space(self) -> int:
        return int(self.doc["subtask"]["target_space"])


def load_workload(name: str, root: str = GOLDEN_DIR) -> Workload:
    d = os.path.join(root, name)
    tn = load_network(os.path.join(d, "network.json"))
    with open(os.path.join(d, "order.json")) as fh:
        doc = json.load(fh)
    return Workload(name=name, tn=tn, tree=doc_to_tree(doc), doc=doc)
