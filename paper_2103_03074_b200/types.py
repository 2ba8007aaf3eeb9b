"""Data types of the drop-in engine API.

``EngineStats``, ``HeadVector`` and ``AmplitudeTable`` are the reference's
own dataclasses (engine.py:44-96) when ``tncut`` is importable, so results
flow into the rest of the reference package (TSV/HV writers, analytics)
unchanged.  Otherwise field-for-field identical definitions are used.

``Step``, ``StepCost`` and ``ContractionTree`` restate the reference's
tree types (ordering.py:31-147) for fixture-driven use without ``tncut``;
the engine itself only duck-types trees (``leaves``, ``steps``,
``first_cut``, ``head_steps()``, ``tail_steps()``, ``head_tail_leaves()``).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np

try:  # pragma: no cover - environment dependent
    from tncut.engine import AmplitudeTable, EngineStats, HeadVector  # type: ignore
except Exception:

    @dataclass
    class EngineStats:  # engine.py:44-49
        multiplications: int = 0
        head_contractions: int = 0
        tail_contractions: int = 0
        steps_executed: int = 0

    @dataclass
    class HeadVector:  # engine.py:52-65
        s1: dict
        data: np.ndarray
        provenance: str
        cut_order: list
        n_e: int
        slice_range: tuple
        mode: str
        sliced_indices: tuple = ()

        @property
        def n_c(self) -> int:
            return len(self.cut_order)

    @dataclass
    class AmplitudeTable:  # engine.py:68-96
        s1: dict
        open_qubits: list
        amplitudes: np.ndarray
        layout_ids: list
        circuit_sha256: str
        order_sha256: str
        precision: str
        mode: str

        @property
        def probabilities(self) -> np.ndarray:
            return np.abs(self.amplitudes) ** 2

        def bitstring(self, mask: int) -> str:
            n2 = len(self.open_qubits)
            s2 = {q: (mask >> (n2 - 1 - i)) & 1 for i, q in enumerate(self.open_qubits)}
            return "".join(str(s2[q] if q in s2 else self.s1[q]) for q in sorted(self.layout_ids))

        def rows(self):
            for mask, amp in enumerate(self.amplitudes):
                yield self.bitstring(mask), complex(amp), float(abs(amp) ** 2)


@dataclass(frozen=True)
class Step:  # ordering.py:31-35
    lhs: int
    rhs: int
    out: int


@dataclass(frozen=True)
class StepCost:  # ordering.py:38-51
    n_a: int
    n_b: int
    n_ab: int
    out_rank: int

    @property
    def time_cost(self) -> int:
        return 1 << (self.n_a + self.n_b + self.n_ab)


@dataclass
class ContractionTree:  # ordering.py:99-147
    leaves: list
    steps: list
    first_cut: int | None = None
    annotations: list | None = None
    seed: int | None = None
    constraints: dict | None = None

    def root_id(self) -> int:
        return self.steps[-1].out if self.steps else self.leaves[0]

    def subtree_leaves(self) -> dict:
        cover = {leaf: frozenset([leaf]) for leaf in self.leaves}
        for s in self.steps:
            cover[s.out] = cover[s.lhs] | cover[s.rhs]
        return cover

    def head_tail_leaves(self):
        if self.first_cut is None:
            return frozenset(), frozenset(self.leaves)
        cover = self.subtree_leaves()
        cut = self.steps[self.first_cut]
        return cover[cut.lhs], cover[cut.rhs]

    def _side_steps(self, root) -> list:
        want = {root}
        picked = []
        for s in reversed(self.steps[: self.first_cut]):
            if s.out in want:
                picked.append(s)
                want.update((s.lhs, s.rhs))
        return picked[::-1]

    def head_steps(self) -> list:
        if self.first_cut is None:
            return []
        return self._side_steps(self.steps[self.first_cut].lhs)

    def tail_steps(self) -> list:
        if self.first_cut is None:
            return list(self.steps)
        return self._side_steps(self.steps[self.first_cut].rhs)


ORDER_SCHEMA = "tncut-order/1"


def tree_to_doc(tree, tn=None, circuit_sha256=None, open_qubits=None, slices=None,
                subtask=None) -> dict:
    """Order document (restates ordering.py:670-707)."""
    doc = {
        "schema": ORDER_SCHEMA,
        "leaves": list(tree.leaves),
        "steps": [{"lhs": s.lhs, "rhs": s.rhs, "out": s.out} for s in tree.steps],
        "first_cut": tree.first_cut,
        "seed": tree.seed,
        "constraints": tree.constraints,
    }
    if tree.annotations is not None:
        doc["annotations"] = [dataclasses.asdict(a) for a in tree.annotations]
        tc = sum(a.time_cost for a in tree.annotations)
        doc["tc"] = tc
        doc["tc_log2"] = math.log2(tc) if tc else 0.0
        doc["sc_log2"] = max((a.out_rank for a in tree.annotations), default=0)
    if circuit_sha256 is not None:
        doc["circuit_sha256"] = circuit_sha256
    if open_qubits is not None:
        doc["open_qubits"] = sorted(open_qubits)
    if slices is not None:
        doc["slices"] = list(slices)
    if subtask is not None:
        doc["subtask"] = subtask
    return doc


def doc_to_tree(doc: dict) -> ContractionTree:
    """Inverse of tree_to_doc (restates ordering.py:710-722)."""
    if doc.get("schema") != ORDER_SCHEMA:
        raise ValueError(f"unknown order schema {doc.get('schema')!r}")
    tree = ContractionTree(
        leaves=list(doc["leaves"]),
        steps=[Step(s["lhs"], s["rhs"], s["out"]) for s in doc["steps"]],
        first_cut=doc.get("first_cut"),
        seed=doc.get("seed"),
        constraints=doc.get("constraints"),
    )
    if "annotations" in doc:
        tree.annotations = [StepCost(**a) for a in doc["annotations"]]
    return tree
