"""numpy restatement of the reference engine -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference lines it follows
(/root/reference/pkg/src/tncut/engine.py unless noted).  Inputs are
duck-typed networks/trees (``nodes[id].indices/.data``, ``index_endpoints``,
``open_output_indices``; ``leaves``, ``steps``, ``first_cut``,
``head_steps()``, ``tail_steps()``, ``head_tail_leaves()``).
"""

from __future__ import annotations

import numpy as np

DTYPES = {"double": np.complex128, "single": np.complex64}


class Stats:
    """engine.py:44-49"""

    def __init__(self):
        self.multiplications = 0
        self.head_contractions = 0
        self.tail_contractions = 0
        self.steps_executed = 0


def prepared_leaves(tn, leaf_ids, assignment, dtype):
    """engine.py:102-114: cast, then np.take each pinned axis."""
    tensors = {}
    for nid in leaf_ids:
        node = tn.nodes[nid]
        data = node.data.astype(dtype, copy=False)
        ids = list(node.indices)
        for ix, bit in assignment.items():
            if ix in ids:
                ax = ids.index(ix)
                data = np.take(data, bit, axis=ax)
                del ids[ax]
        tensors[nid] = (data, ids)
    return tensors


def contract_steps(tn, leaf_ids, steps, assignment, dtype, stats=None, extra=None):
    """engine.py:117-144: pairwise tensordot / outer product.

    ``extra``: optional {id: (data, ids)} leaves not in ``tn`` (used by the
    head-absorbed tail)."""
    tensors = prepared_leaves(tn, leaf_ids, assignment, dtype)
    if extra:
        tensors.update({k: (np.asarray(v[0], dtype=dtype), list(v[1])) for k, v in extra.items()})
    for s in steps:
        lhs, rhs, out = (s.lhs, s.rhs, s.out) if hasattr(s, "lhs") else s
        a, a_ids = tensors.pop(lhs)
        b, b_ids = tensors.pop(rhs)
        shared = [ix for ix in a_ids if ix in b_ids]
        if shared:
            ax_a = [a_ids.index(ix) for ix in shared]
            ax_b = [b_ids.index(ix) for ix in shared]
            res = np.tensordot(a, b, axes=(ax_a, ax_b))
        else:
            res = np.multiply.outer(a, b)
        out_ids = [ix for ix in a_ids if ix not in b_ids] + [ix for ix in b_ids if ix not in a_ids]
        assert res.ndim == len(out_ids)
        tensors[out] = (res, out_ids)
        if stats is not None:
            stats.multiplications += 1 << (len(a_ids) + len(b_ids) - len(shared))
            stats.steps_executed += 1
    assert len(tensors) == 1, f"{len(tensors)} results left"
    (tensor, ids), = tensors.values()
    return tensor, ids


def contract_tree(tn, tree, assignment, dtype=np.complex128, stats=None):
    """engine.py:147-165: root axes sorted by index id."""
    tensor, ids = contract_steps(tn, tree.leaves, tree.steps, assignment, dtype, stats)
    if ids:
        tensor = np.transpose(tensor, sorted(range(len(ids)), key=lambda k: ids[k]))
    return tensor


def cut_indices(tn, head, tail):
    """ordering.py:372-380"""
    out = []
    for ix, eps in tn.index_endpoints.items():
        if len(eps) == 2:
            inh = [e in head for e in eps]
            if any(inh) and not all(inh):
                out.append(ix)
    return sorted(out)


def split(tn, tree):
    """engine.py:171-185"""
    if tree.first_cut is not None:
        h, t = tree.head_tail_leaves()
        return sorted(h), tree.head_steps(), sorted(t), tree.tail_steps(), cut_indices(tn, set(h), set(t))
    if tn.open_output_indices:
        return [], [], sorted(tree.leaves), list(tree.steps), []
    return sorted(tree.leaves), list(tree.steps), [], [], []


def fixed_tree_sum(chunks):
    """engine.py:207-222: balanced binary-counter summation."""
    stack = []
    for x in chunks:
        level = 0
        while stack and stack[-1][0] == level:
            _, prev = stack.pop()
            x = prev + x
            level += 1
        stack.append((level, x))
    if not stack:
        return None
    total = stack[0][1]
    for _, part in stack[1:]:
        total = total + part
    return total


def head_vector(tn, tree, sliced, slice_range=None, precision="single", mode="fixed", stats=None):
    """engine.py:242-310 (data only; tn must already be pinned to s1)."""
    head_leaves, head_steps, _, _, cut = split(tn, tree)
    n_e = len(sliced)
    a, b = slice_range if slice_range is not None else (0, 1 << n_e)
    dtype = DTYPES[precision]

    def head_result(mask):
        assignment = {ix: (mask >> (n_e - 1 - pos)) & 1 for pos, ix in enumerate(sliced)}
        if stats is not None:
            stats.head_contractions += 1
        if not head_leaves:
            return np.ones(1, dtype=dtype)
        tensor, ids = contract_steps(tn, head_leaves, head_steps, assignment, dtype, stats)
        order = [ids.index(ix) for ix in sorted(cut)]
        return np.transpose(tensor, order).reshape(-1)

    chunks = (head_result(m) for m in range(a, b))
    if mode == "fixed":
        return fixed_tree_sum(chunks)
    data = None
    for x in chunks:
        data = x if data is None else data + x
    return data


def tail_blocked(tn, tree, head_data, space_cap=None, precision="single", stats=None):
    """engine.py:313-378 (reference-faithful blocked tail, no provenance)."""
    _, _, tail_leaves, tail_steps, cut = split(tn, tree)
    dtype = DTYPES[precision]
    opens = sorted(tn.open_output_indices)
    n2, n_c = len(opens), len(cut)
    amps = np.zeros(1 << n2, dtype=dtype)
    if not tail_leaves:
        amps[0] = head_data[0]
        return amps
    k = 0
    if space_cap is not None:
        while n2 - k + n_c > space_cap and k < n2:
            k += 1
    pinned, free = opens[:k], opens[k:]
    free_ixs = [tn.open_output_indices[q] for q in free]
    hd = np.asarray(head_data).astype(dtype, copy=False)
    for block in range(1 << k):
        asg = {tn.open_output_indices[q]: (block >> (k - 1 - i)) & 1 for i, q in enumerate(pinned)}
        if stats is not None:
            stats.tail_contractions += 1
        tensor, ids = contract_steps(tn, tail_leaves, tail_steps, asg, dtype, stats)
        want = free_ixs + sorted(cut)
        tensor = np.transpose(tensor, [ids.index(ix) for ix in want]).reshape(1 << len(free), 1 << n_c)
        ba = tensor @ hd
        if stats is not None:
            stats.multiplications += 1 << (len(free) + n_c)
        amps[block << len(free): (block << len(free)) + ba.size] = ba
    return amps


def greedy_steps(sets, next_out):
    """ordering.py:256-285 (deterministic greedy pair order)."""
    sets = {k: frozenset(v) for k, v in sets.items()}
    live = sorted(sets)
    steps = []

    def key(i, j):
        a, b = sets[i], sets[j]
        return (len(a ^ b), len(a | b), i, j)

    pairs = {(i, j): key(i, j) for x, i in enumerate(live) for j in live[x + 1:]}
    while len(live) > 1:
        i, j = min(pairs, key=lambda p: pairs[p])
        out = next_out
        next_out += 1
        sets[out] = sets[i] ^ sets[j]
        steps.append((i, j, out))
        live.remove(i)
        live.remove(j)
        for p in [p for p in pairs if i in p or j in p]:
            del pairs[p]
        for o in live:
            pairs[(o, out) if o < out else (out, o)] = key(*((o, out) if o < out else (out, o)))
        live.append(out)
    return steps


def tail_absorbed(tn, tree, head_data, precision="single"):
    """Head vector absorbed as a leaf; greedy order; open qubits ascending, MSB first.

    Same contraction as engine.py:358-377 summed over blocks (the block
    GEMV is a contraction over the cut indices)."""
    _, _, tail_leaves, _, cut = split(tn, tree)
    dtype = DTYPES[precision]
    hid = max(tn.nodes) + 1
    sets = {nid: tn.nodes[nid].indices for nid in tail_leaves}
    sets[hid] = list(cut)
    steps = greedy_steps(sets, hid + 1)
    head = np.asarray(head_data, dtype=dtype).reshape((2,) * len(cut))
    tensor, ids = contract_steps(tn, tail_leaves, steps, {}, dtype,
                                 extra={hid: (head, list(cut))})
    opens = sorted(tn.open_output_indices)
    order = [ids.index(tn.open_output_indices[q]) for q in opens]
    return np.transpose(tensor, order).reshape(-1)


def combine_partials(parts):
    """engine.py:428-447 on [(range, data)] covering [0, total)."""
    parts = sorted(parts, key=lambda p: p[0][0])
    total = parts[-1][0][1]

    def comb(lo, hi, items):
        if len(items) == 1 and items[0][0] == (lo, hi):
            return items[0][1]
        mid = (lo + hi) // 2
        left = [p for p in items if p[0][1] <= mid]
        right = [p for p in items if p[0][0] >= mid]
        if len(left) + len(right) == len(items) and left and right:
            return comb(lo, mid, left) + comb(mid, hi, right)
        acc = items[0][1]
        for p in items[1:]:
            acc = acc + p[1]
        return acc

    return comb(0, total, parts)


def xeb(probs, n):
    """analytics.py:46-58: F = 2^n/L * sum(p) - 1."""
    probs = np.asarray(probs, dtype=float)
    return (2.0 ** n / probs.size) * float(probs.sum()) - 1.0
