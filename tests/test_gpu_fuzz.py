"""Randomised contraction-program parity (GPU): random tensor networks with
random axis orders, random pairwise orders and random sliced bonds, with the
tensor-core threshold lowered (TNB_TC_MIN_RANK) so that most steps run on
tcgen05 and most step->step edges use fused operand staging (the epilogue
writing the consumer's fp16 layout through the planned bit permutations).
Checked against one np.einsum of the whole network in complex128."""

from __future__ import annotations

import string

import numpy as np
import pytest

from conftest import rel_l2


def _random_network(rng, n_t=None):
    n_t = int(rng.integers(4, 7)) if n_t is None else n_t
    nxt = [100]

    def new():
        nxt[0] += 1
        return nxt[0]

    inds = [[] for _ in range(n_t)]
    bonds = []
    for i in range(n_t - 1):  # chain bonds
        for _ in range(int(rng.integers(3, 6))):
            x = new()
            inds[i].append(x)
            inds[i + 1].append(x)
            bonds.append(x)
    for _ in range(2):  # cross bonds
        i, j = sorted(rng.choice(n_t, 2, replace=False))
        x = new()
        inds[i].append(x)
        inds[j].append(x)
        bonds.append(x)
    opens = []
    for i in range(n_t):
        for _ in range(int(rng.integers(2, 5))):
            x = new()
            inds[i].append(x)
            opens.append(x)
    leaves = []
    for i in range(n_t):
        ix = list(rng.permutation(inds[i]))
        data = (rng.standard_normal(1 << len(ix)) + 1j * rng.standard_normal(1 << len(ix))) / 2
        leaves.append((i + 1, [int(v) for v in ix], data.reshape((2,) * len(ix))))
    # random pairwise order, preferring pairs that share an index
    live = {nid: set(ix) for nid, ix, _ in leaves}
    steps, out_id = [], 1000
    while len(live) > 1:
        keys = sorted(live)
        pairs = [(a, b) for x, a in enumerate(keys) for b in keys[x + 1:] if live[a] & live[b]]
        a, b = pairs[int(rng.integers(len(pairs)))] if pairs else (keys[0], keys[1])
        if rng.random() < 0.5:
            a, b = b, a
        live[out_id] = live.pop(a) ^ live.pop(b)
        steps.append((a, b, out_id))
        out_id += 1
    sliced = [int(v) for v in rng.choice(bonds, size=int(rng.integers(0, 3)), replace=False)]
    # keep every tensor <= 2^24 entries (the einsum check runs on the host)
    live = {nid: set(ix) for nid, ix, _ in leaves}
    for a, b, o in steps:
        live[o] = live.pop(a) ^ live.pop(b)
        if len(live[o]) > 24:
            return _random_network(rng)
    if len(bonds) + len(opens) > 52 or any(len(ix) > 20 for _, ix, _ in leaves):
        return _random_network(rng)
    return leaves, steps, sliced, sorted(opens)


def _einsum(leaves, out_order):
    letters = {}
    pool = iter(string.ascii_letters)
    terms = []
    for _, ix, _ in leaves:
        for i in ix:
            if i not in letters:
                letters[i] = next(pool)
        terms.append("".join(letters[i] for i in ix))
    spec = ",".join(terms) + "->" + "".join(letters[i] for i in out_order)
    return np.einsum(spec, *[d.astype(np.complex128) for _, _, d in leaves], optimize=True)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
def test_random_networks_tensor_core_and_fused_paths(gpu, seed, monkeypatch):
    from paper_2103_03074_b200 import _lib
    from paper_2103_03074_b200.engine import Program

    rng = np.random.default_rng(seed)
    leaves, steps, sliced, opens = _random_network(rng)
    ref = _einsum(leaves, opens).reshape(-1)
    n_masks = 1 << len(sliced)
    results = {}
    for name, env, flags in (("fused", "14", 0), ("staged", "14", _lib.TNB_FLAG_NO_FUSE),
                             ("simt", "99", 0)):
        monkeypatch.setenv("TNB_TC_MIN_RANK", env)
        prog = Program(leaves, steps, sliced, opens, "single", 0, flags)
        if name == "fused":
            assert prog.info.n_steps_tc >= 1
            fused = prog.info.n_steps_fused
        results[name] = prog.run_range(0, n_masks, "fixed")
        del prog
    for name, got in results.items():
        err = rel_l2(got, ref)
        assert err < 1e-4, (name, err, fused)
    # tensor-core paths agree with the fp32 SIMT path to fp32-level accuracy
    assert rel_l2(results["fused"], results["simt"]) < 1e-5


@pytest.mark.gpu
def test_random_networks_exercise_fusion(gpu, monkeypatch):
    """The generator really produces fused edges (else the test above would
    only cover the staged path)."""
    from paper_2103_03074_b200.engine import Program

    monkeypatch.setenv("TNB_TC_MIN_RANK", "14")
    total_fused = 0
    for seed in range(10):
        leaves, steps, sliced, opens = _random_network(np.random.default_rng(seed))
        prog = Program(leaves, steps, sliced, opens, "single", 0, 0)
        total_fused += prog.info.n_steps_fused
        del prog
    assert total_fused >= 5, total_fused


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_random_networks_slice_blocks(gpu, seed, monkeypatch):
    """Batched slices at program level (slice_batch.py's principle): the plan
    with the LAST k sliced indices un-sliced, mask j, equals the full plan's
    masks [j*2^k, (j+1)*2^k) summed (engine.py:276-279 mask convention)."""
    from paper_2103_03074_b200.engine import Program

    rng = np.random.default_rng(1000 + seed)
    for _ in range(50):
        leaves, steps, sliced, opens = _random_network(rng)
        if len(sliced) >= 2:
            break
    else:
        pytest.skip("no network with two sliced bonds")
    monkeypatch.setenv("TNB_TC_MIN_RANK", "14")
    full = Program(leaves, steps, sliced, opens, "single", 0, 0)
    k = 1
    blk = Program(leaves, steps, sliced[: len(sliced) - k], opens, "single", 0, 0)
    for j in range(1 << (len(sliced) - k)):
        want = full.run_range(j << k, (j + 1) << k, "fixed")
        got = blk.run_range(j, j + 1, "fixed")
        assert rel_l2(got, want) < 1e-5, (j, rel_l2(got, want))
