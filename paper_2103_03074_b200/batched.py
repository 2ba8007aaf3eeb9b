"""Batched closed-bit assignments: several s1 values
that share one contraction tree, contracted in ONE pass.

The reference computes one head vector per s1 (``compute_head_vector``,
engine.py:242-310; ``TensorNetwork.repin``, network.py:65-77).  Assignments
that differ only in a few closed qubits Q differ only in the projection
tensors of those qubits' output legs.  Keeping those legs open (a dangling
index per qubit of Q) gives one network whose head contraction yields all
2^|Q| head vectors at once; the tree stays valid (same node ids, the extra
indices never contract and ride up to the head root).  On the C4 plan one
such qubit adds ~2 % of head work for twice the assignments (4 qubits:
16 assignments for 1.25x), so the correlated-bitstring batch grows almost
for free.

The un-pinned tensors are rebuilt from the network's own ``repin`` (both
bit values of each qubit, stacked along a fresh index), so this works for
the reference's ``TensorNetwork`` and the frozen workloads alike.  The
result is a list of ordinary ``HeadVector`` objects, one per requested s1,
numerically the per-s1 results (parity: tests/test_batched.py).
"""

from __future__ import annotations

import dataclasses
import itertools

import numpy as np

from . import engine as E
from .errors import RangeOutOfBounds, ShapeMismatch
from .planner import split
from .provenance import normalize_s1, provenance_hash
from .types import HeadVector


def _replace_nodes(tn, new_nodes: dict):
    """The network with some nodes replaced (duck-typed dataclass copy)."""
    nodes = dict(tn.nodes)
    nodes.update(new_nodes)
    out = dataclasses.replace(tn, nodes=nodes) if dataclasses.is_dataclass(tn) else tn
    eps: dict = {}
    for node in nodes.values():
        for ix in node.indices:
            eps.setdefault(ix, []).append(node.id)
    out.index_endpoints = {ix: tuple(v) for ix, v in eps.items()}
    return out


def batched_network(tn, s1_list):
    """(network with the varying closed qubits' legs open, varying qubits in
    order, their new index ids, the shared base assignment)."""
    s1s = [normalize_s1(tn, s) for s in s1_list]
    if not s1s:
        raise ValueError("no assignments given")
    closed = sorted(s1s[0])
    qs = [q for q in closed if len({s[q] for s in s1s}) > 1]
    base = dict(s1s[0])
    ref = tn.repin(base)
    if not qs:
        return ref, [], [], base, s1s
    next_ix = 1 + max(ix for node in ref.nodes.values() for ix in node.indices)
    q_ix = {}
    # which node carries each qubit's projection: the one that changes with it
    owner = {}
    for q in qs:
        flip = dict(base)
        flip[q] = 1 - base[q]
        other = tn.repin(flip)
        diff = [nid for nid in ref.nodes
                if not np.array_equal(np.asarray(ref.nodes[nid].data), np.asarray(other.nodes[nid].data))]
        if len(diff) != 1:
            raise ShapeMismatch(f"closed qubit {q}: {len(diff)} nodes depend on its bit")
        owner[q] = diff[0]
        q_ix[q] = next_ix
        next_ix += 1
    new_nodes = {}
    for nid in sorted(set(owner.values())):
        mine = [q for q in qs if owner[q] == nid]
        node = ref.nodes[nid]
        # stack the node over every assignment of its qubits: new axes first
        # (in `mine` order, MSB first), then the node's own axes
        blocks = []
        for bits in itertools.product((0, 1), repeat=len(mine)):
            asg = dict(base)
            asg.update(zip(mine, bits))
            blocks.append(np.asarray(tn.repin(asg).nodes[nid].data))
        data = np.stack(blocks).reshape((2,) * len(mine) + tuple(np.shape(blocks[0])))
        new_nodes[nid] = dataclasses.replace(node, indices=[q_ix[q] for q in mine] + list(node.indices),
                                             data=np.ascontiguousarray(data))
    return _replace_nodes(ref, new_nodes), qs, [q_ix[q] for q in qs], base, s1s


def compute_head_vectors_batched(tn, tree, sliced_indices, s1_list, slice_range=None,
                                 precision="double", mode="fixed", stats=None, device=None):
    """One HeadVector per entry of ``s1_list`` (same meaning as calling
    ``compute_head_vector`` per s1), from a single contraction of the
    network with the varying closed qubits' output legs kept open."""
    tnb, qs, q_ix, base, s1s = batched_network(tn, s1_list)
    sliced_indices = list(sliced_indices)
    head_leaves, head_steps, _, _, cut = split(tnb, tree)
    head_set = set(head_leaves)
    for ix in sliced_indices:
        eps = tnb.index_endpoints.get(ix, ())
        if len(eps) != 2 or any(e not in head_set for e in eps):
            raise ShapeMismatch(f"sliced index {ix} is not internal to the head")
    for ix in q_ix:
        if tnb.index_endpoints.get(ix, ())[0] not in head_set:
            raise ShapeMismatch("a varying closed qubit's node is not in the head")
    n_e = len(sliced_indices)
    total = 1 << n_e
    a, b = slice_range if slice_range is not None else (0, total)
    if not (0 <= a < b <= total):
        raise RangeOutOfBounds(f"range [{a},{b}) outside [0,{total})")
    cut = sorted(cut)
    # root axes: the varying qubits (major, MSB first), then the cut ids
    entries = E._leaf_entries(tnb, head_leaves)
    prog = E.get_program(entries, E._steps_tuples(head_steps), sliced_indices, list(q_ix) + cut,
                         precision, device, upload=False)
    data = prog.run(entries, a, b, mode)
    if stats is not None:
        from .planner import step_mults

        sets = {nid: tnb.nodes[nid].indices for nid in head_leaves}
        mults, _ = step_mults(sets, head_steps, frozenset(sliced_indices))
        stats.multiplications += mults * (b - a)
        stats.head_contractions += (b - a)
        stats.steps_executed += len(head_steps) * (b - a)
    n_c = len(cut)
    block = data.reshape((1 << len(qs), 1 << n_c))
    out = []
    for s in s1s:
        j = 0
        for q in qs:
            j = (j << 1) | int(s[q])
        out.append(HeadVector(
            s1=s, data=np.array(block[j]),
            provenance=provenance_hash(tn, tree, s, precision, mode, sliced_indices),
            cut_order=cut, n_e=n_e, slice_range=(a, b), mode=mode,
            sliced_indices=tuple(sliced_indices)))
    return out


def cheapest_batch_qubits(tn, tree, sliced_indices, b: int):
    """Closed qubits whose un-pinned output legs add the least head work
    (exact multiplication counts of the head schedule, planner.step_mults),
    greedily, b of them.  Returns (qubits, cost ratio vs one assignment)."""
    from .planner import step_mults

    base = tn.repin(dict(tn.fixed_output_bits))
    head_leaves, head_steps, _, _, _ = split(base, tree)
    sl = frozenset(sliced_indices)
    sets = {nid: list(base.nodes[nid].indices) for nid in head_leaves}
    m0, _ = step_mults(sets, head_steps, sl)
    chosen, cur = [], dict(sets)
    nxt = 1 + max(ix for v in sets.values() for ix in v)
    owners = {}
    for q in sorted(tn.fixed_output_bits):
        flip = dict(tn.fixed_output_bits)
        flip[q] = 1 - flip[q]
        other = tn.repin(flip)
        diff = [nid for nid in head_leaves
                if not np.array_equal(np.asarray(base.nodes[nid].data), np.asarray(other.nodes[nid].data))]
        if len(diff) == 1:
            owners[q] = diff[0]
    ratio = 1.0
    for _ in range(b):
        best = None
        for q, nid in owners.items():
            if q in chosen:
                continue
            trial = dict(cur)
            trial[nid] = cur[nid] + [nxt]
            m, _ = step_mults(trial, head_steps, sl)
            if best is None or m < best[0]:
                best = (m, q, trial)
        if best is None:
            break
        ratio = best[0] / m0
        chosen.append(best[1])
        cur = best[2]
        nxt += 1
    return chosen, ratio
