"""Provenance bookkeeping restated from the reference engine.

``provenance_hash`` (engine.py:188-204) and ``normalize_s1``
(engine.py:225-239) are re-implemented so the drop-in needs no ``tncut``
import at run time; tests check both against the reference here.
"""

from __future__ import annotations

import hashlib
import weakref
import json

from .errors import ProvenanceMismatch
from .types import tree_to_doc


def dumps_order(doc: dict) -> str:
    """Canonical order-document text (ordering.py:720-721)."""
    return json.dumps(doc, sort_keys=True, separators=(",", ":")) + "\n"


def circuit_sha(tn) -> str:
    return tn.circuit.sha256() if getattr(tn, "circuit", None) is not None else "none"


_order_cache: dict = {}


def order_sha256(tree, tn, sliced_indices) -> str:
    """sha256 of the canonical order document; memoised per tree object
    (serialising ~800 steps costs milliseconds per engine call)."""
    csha = circuit_sha(tn)
    sl = tuple(sliced_indices)
    ann = getattr(tree, "annotations", None)
    fp = (len(tree.steps), tree.first_cut, id(tree.steps), id(ann), len(ann or ()), csha, sl,
          getattr(tree, "seed", None))
    hit = _order_cache.get(id(tree))
    if hit is not None and hit[0]() is tree and hit[1] == fp:
        return hit[2]
    doc = tree_to_doc(tree, circuit_sha256=csha, slices=list(sl))
    digest = hashlib.sha256(dumps_order(doc).encode()).hexdigest()
    try:
        if len(_order_cache) > 64:
            _order_cache.clear()
        _order_cache[id(tree)] = (weakref.ref(tree), fp, digest)
    except TypeError:  # not weak-referenceable: no memo
        pass
    return digest


def provenance_hash(tn, tree, s1: dict, precision: str, mode: str, sliced_indices=()) -> str:
    """sha256(circuit sha | order-doc sha | s1 | precision | mode) (engine.py:188-204)."""
    csha = circuit_sha(tn)
    s1_str = "".join(str(s1[q]) for q in sorted(s1)) or "-"
    payload = "|".join([csha, order_sha256(tree, tn, sliced_indices), s1_str, precision, mode])
    return hashlib.sha256(payload.encode()).hexdigest()


def normalize_s1(tn, s1) -> dict:
    """Closed-qubit bit assignment as a dict (engine.py:225-239)."""
    closed = sorted(tn.fixed_output_bits)
    if s1 is None:
        return dict(tn.fixed_output_bits)
    if isinstance(s1, str):
        if s1 == "-" and not closed:
            return {}
        if len(s1) != len(closed):
            raise ProvenanceMismatch(f"s1 has {len(s1)} bits but {len(closed)} qubits are closed")
        return {q: int(b) for q, b in zip(closed, s1)}
    if set(s1) != set(closed):
        raise ProvenanceMismatch("s1 must cover exactly the closed qubits")
    return {q: int(b) for q, b in s1.items()}
