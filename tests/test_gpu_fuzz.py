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

from conftest import rel_l2, measured


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
    assert measured(rel_l2(results["fused"], results["simt"])) < 1e-5


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
        assert measured(rel_l2(got, want)) < 1e-5, (j, rel_l2(got, want))


def _loose_bound_network(rng, huge_log2=13):
    """T1[m,k] T2[k,n] -> X (fused into the next step) then X T3[n,p].
    T1 has one huge entry in column k=0 where T2's row is zero, T2 one huge
    entry in row k=1 where T1's column is zero: the a-priori bound
    2K max|T1| max|T2| of X is ~2^(2*huge_log2+7) while |X| stays O(10) --
    the fused fp16 operand of the second step would sit ~28 binary orders
    below its scale, i.e. in fp16's subnormal range."""
    m, k, n, p = [list(range(100 + 10 * i, 100 + 10 * i + w)) for i, w in enumerate((8, 6, 7, 8))]
    big = float(2 ** huge_log2)

    def rnd(*shape):
        x = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / 2
        return x.astype(np.complex64).astype(np.complex128)  # exactly representable in fp32

    t1 = rnd(1 << 8, 1 << 6)
    t1[:, 1] = 0
    t1[0, 0] = big
    t2 = rnd(1 << 6, 1 << 7)
    t2[0, :] = 0
    t2[1, 0] = big
    t3 = rnd(1 << 7, 1 << 8)
    leaves = [(1, m + k, t1.reshape((2,) * 14)), (2, k + n, t2.reshape((2,) * 13)),
              (3, n + p, t3.reshape((2,) * 15))]
    return leaves, [(1, 2, 1000), (1000, 3, 1001)], m + p


@pytest.mark.gpu
def test_fp16_scale_guard_fires_on_loose_bound(gpu, monkeypatch):
    """The fused operand's fp16 scale comes from an a-priori bound; when the
    result is ~2^-28 of it, the guard re-runs the producer with the exact max
    (timing().scale_redos counts it) and the result stays at fp32 accuracy.
    With the guard off the same program loses accuracy -- the guard is what
    keeps it."""
    from paper_2103_03074_b200.engine import Program

    rng = np.random.default_rng(7)
    leaves, steps, opens = _loose_bound_network(rng)
    ref = _einsum(leaves, opens).reshape(-1)
    monkeypatch.setenv("TNB_TC_MIN_RANK", "14")
    errs = {}
    for name, bits in (("guard", None), ("off", "-1")):
        if bits is None:
            monkeypatch.delenv("TNB_SCALE_GUARD_BITS", raising=False)
        else:
            monkeypatch.setenv("TNB_SCALE_GUARD_BITS", bits)
        prog = Program(leaves, steps, [], opens, "single", 0, 0)
        assert prog.info.n_steps_fused >= 1, "network did not produce a fused edge"
        prog.set_timing(2)
        got = prog.run_range(0, 1, "fixed")
        errs[name] = rel_l2(got, ref)
        redos = prog.timing()["scale_redos"]
        if name == "guard":
            assert redos >= 1
        else:
            assert redos == 0
        del prog
    measured(errs["guard"])
    measured(errs["off"], "control_rel_l2_guard_off")  # negative control: the guard is what fixes it
    assert errs["guard"] < 1e-5, errs
    assert errs["off"] > 10 * errs["guard"], errs


@pytest.mark.gpu
def test_fp16_scale_guard_quiet_on_c2(gpu, workloads):
    """On a real plan (c2, 249 steps) the guard does not fire at its default
    threshold: no re-runs, so the fast path is unchanged."""
    from paper_2103_03074_b200 import engine as E

    w = workloads("c2")
    prog = E.head_program(w.tn, w.tree, w.sliced, "single")
    prog.set_timing(2)
    prog.run_range(0, 2, "fixed")
    t = prog.timing()
    assert prog.info.n_steps_fused >= 1
    assert t["scale_redos"] == 0, t
