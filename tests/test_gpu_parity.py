"""Parity of the CUDA path (through the C-ABI) -- needs a B200.

Bars (BASELINE.json north_star): bitstring selection/indexing bit-exact,
amplitudes within 1e-4 relative L2 (single), XEB within 1e-3 absolute.
Double precision runs the SIMT fp64 path: 1e-10 relative.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import golden, rel_l2, measured
from oracle import engine_np as O

pytestmark = pytest.mark.gpu

SINGLE_TOL = 1e-4


def _cgemm(lib, M, N, K, use_tc, seed=0):
    from paper_2103_03074_b200 import _lib

    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))).astype(np.complex64)
    B = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    Cm = np.empty((M, N), dtype=np.complex64)
    _lib.check(lib.tnb_cgemm(0, M, N, K, A.ctypes.data, B.ctypes.data, Cm.ctypes.data, 0,
                             1 if use_tc else 0))
    ref = A.astype(np.complex128) @ B.astype(np.complex128)
    return Cm, ref, A, B


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 128, 128), (1024, 512, 256),
                                   (4096, 256, 1024), (128, 4096, 512), (512, 64, 8192),
                                   (8192, 2048, 64), (64, 64, 65536),
                                   # K-blocked layout boundaries: 2K = 16, 32 (one partial /
                                   # exact K block, row-major) and 64 (first blocked size);
                                   # N = 8 (16 expanded columns of a 256-wide tile)
                                   (256, 8, 8), (128, 16, 16), (512, 256, 32), (2048, 8, 4096)])
def test_cgemm_tensor_core_vs_fp64(gpu, M, N, K):
    Cm, ref, A, B = _cgemm(gpu, M, N, K, True)
    err = rel_l2(Cm, ref)
    # the fp32 floor of a length-K dot product
    c64 = A @ B
    assert err < max(4 * rel_l2(c64, ref), 2e-6), (err, rel_l2(c64, ref))


def test_cgemm_simt_vs_fp64(gpu):
    Cm, ref, _, _ = _cgemm(gpu, 64, 32, 128, False)
    assert measured(rel_l2(Cm, ref)) < 1e-6


def test_cgemm_scaled_inputs(gpu):
    """Tiny magnitudes (amplitude-like, ~2^-26) survive the fp16 split scaling."""
    from paper_2103_03074_b200 import _lib

    rng = np.random.default_rng(3)
    M = N = K = 256
    A = ((rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))) * 2.0 ** -26).astype(np.complex64)
    B = ((rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))) * 2.0 ** 20).astype(np.complex64)
    Cm = np.empty((M, N), dtype=np.complex64)
    _lib.check(gpu.tnb_cgemm(0, M, N, K, A.ctypes.data, B.ctypes.data, Cm.ctypes.data, 0, 1))
    assert measured(rel_l2(Cm, A.astype(np.complex128) @ B.astype(np.complex128))) < 2e-6


# ---------------------------------------------------------------------------
# C1: 3x4 grid, all 2^12 amplitudes vs the state vector

@pytest.mark.parametrize("precision", ["double", "single"])
def test_c1_all_amplitudes(gpu, workloads, precision):
    w = workloads("c1")
    g = golden("c1")
    closed = sorted(w.tn.fixed_output_bits)
    amps = []
    for s1v in range(256):
        s1 = "".join(str((s1v >> (len(closed) - 1 - i)) & 1) for i in range(len(closed)))
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s1, precision=precision)
        tab = tnb.compute_tail_amplitudes(w.tn, w.tree, hv, space_cap=8, precision=precision)
        amps.append(tab.amplitudes)
    amps = np.array(amps)
    tol = 1e-10 if precision == "double" else SINGLE_TOL
    assert measured(rel_l2(amps, g["amps_statevector"])) < tol
    # total probability over all 2^12 bitstrings
    assert abs(np.sum(np.abs(amps.astype(np.complex128)) ** 2) - 1.0) < (1e-9 if precision == "double" else 1e-4)


def test_c1_head_matches_reference_double(gpu, workloads):
    w = workloads("c1")
    g = golden("c1")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="double")
    assert measured(rel_l2(hv.data, g["head_full_double"])) < 1e-12
    assert hv.provenance == str(g["provenance"])
    assert hv.cut_order == sorted(hv.cut_order)


@pytest.mark.parametrize("mode", ["fixed", "free"])
def test_c1_ranges(gpu, workloads, mode):
    w = workloads("c1")
    g = golden("c1")
    for (a, b) in [(0, 8), (8, 16), (3, 11)]:
        p = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(a, b),
                                    precision="double", mode=mode)
        assert p.slice_range == (a, b)
        assert measured(rel_l2(p.data, g[f"head_{mode}_{a}_{b}"])) < 1e-12


@pytest.mark.parametrize("precision", ["double", "single"])
def test_fixed_mode_partials_reduce_bit_exactly(gpu, workloads, precision):
    """Aligned power-of-two partials recombine to the single-shot result bit-for-bit."""
    w = workloads("c1")
    full = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision=precision)
    parts = [tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(a, a + 4),
                                     precision=precision) for a in (12, 0, 4, 8)]
    red = tnb.reduce_partials(parts)
    assert red.slice_range == (0, 16)
    assert np.array_equal(red.data, full.data)


def test_c1_stats_match_reference(gpu, workloads):
    w = workloads("c1")
    g = golden("c1")
    st = tnb.EngineStats()
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="double", stats=st)
    assert [st.multiplications, st.head_contractions, st.steps_executed] == \
        [int(g["head_stats"][0]), int(g["head_stats"][1]), int(g["head_stats"][3])]
    st2 = tnb.EngineStats()
    tnb.compute_tail_amplitudes(w.tn, w.tree, hv, space_cap=6, precision="double", stats=st2)
    assert [st2.multiplications, st2.tail_contractions, st2.steps_executed] == \
        [int(g["tail_stats_cap6"][0]), int(g["tail_stats_cap6"][2]), int(g["tail_stats_cap6"][3])]


def test_c1_contract_tree(gpu, workloads):
    w = workloads("c1")
    g = golden("c1")
    asg = {ix: (5 >> (w.n_e - 1 - p)) & 1 for p, ix in enumerate(w.sliced)}
    out = tnb.contract_tree(w.tn, w.tree, asg)
    assert out.shape == g["contract_tree_mask5"].shape
    assert measured(rel_l2(out, g["contract_tree_mask5"])) < 1e-12


def test_errors(gpu, workloads):
    w = workloads("c1")
    with pytest.raises(tnb.RangeOutOfBounds):
        tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 17))
    with pytest.raises(tnb.RangeOutOfBounds):
        tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(5, 5))
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 8))
    with pytest.raises(tnb.ProvenanceMismatch):
        tnb.compute_tail_amplitudes(w.tn, w.tree, hv)
    full = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision="single")
    with pytest.raises(tnb.ProvenanceMismatch):
        tnb.compute_tail_amplitudes(w.tn, w.tree, full, precision="double")
    with pytest.raises(ValueError):
        tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, mode="bogus")
    # a tail/cut index is not head-internal
    bad = list(w.sliced) + [w.tn.open_output_indices[min(w.tn.open_output_indices)]]
    with pytest.raises(tnb.ShapeMismatch):
        tnb.compute_head_vector(w.tn, w.tree, bad, None)
    with pytest.raises(tnb.RangeGap):
        tnb.reduce_partials([hv])


# ---------------------------------------------------------------------------
# Sycamore-53 configs against the oracle / reference goldens

def _head_vs_golden(w, g, rng_, precision="single"):
    a, b = rng_
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=rng_,
                                 precision=precision)
    stride = int(g["stride"])
    key = f"head_{precision}_{a}_{b}"
    err = rel_l2(hv.data[::stride], g[key + "_sub"])
    norm_ratio = float(np.vdot(hv.data, hv.data).real) / float(g[key + "_norm2"])
    return hv, err, norm_ratio


def test_s8_head_and_tail(gpu, workloads):
    w = workloads("s8")
    g = golden("s8")
    hv, err, nr = _head_vs_golden(w, g, (0, 4))
    assert err < SINGLE_TOL and abs(nr - 1) < 2 * SINGLE_TOL
    _, errd, _ = _head_vs_golden(w, g, (0, 4), "double")
    assert errd < 1e-10
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    assert measured(rel_l2(tab.amplitudes, g["amps_sub"])) < SINGLE_TOL
    # oracle at full size, same inputs
    ref = O.head_vector(w.tn, w.tree, w.sliced, (0, 4), "single")
    assert measured(rel_l2(hv.data, ref)) < SINGLE_TOL


def test_s8_fixed_vs_free_and_ranges(gpu, workloads):
    w = workloads("s8")
    ref = O.head_vector(w.tn, w.tree, w.sliced, (4, 12), "single", "free")
    for mode in ("fixed", "free"):
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(4, 12),
                                     precision="single", mode=mode)
        assert measured(rel_l2(hv.data, ref)) < SINGLE_TOL


@pytest.mark.parametrize("name", ["m12", "c2", "c4"])
def test_sycamore_head_slice_vs_reference(gpu, workloads, name):
    """One head slice at the BASELINE plans (tensor-core GEMM steps)."""
    w = workloads(name)
    g = golden(name)
    hv, err, nr = _head_vs_golden(w, g, (0, 1))
    assert err < SINGLE_TOL, err
    assert abs(nr - 1) < 2 * SINGLE_TOL
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    stride = int(g["amps_stride"])
    assert measured(rel_l2(tab.amplitudes[::stride], g["amps_sub"])) < SINGLE_TOL
    probs = np.abs(tab.amplitudes.astype(np.complex128)) ** 2
    assert abs(probs.sum() / float(g["amps_probsum"]) - 1) < 2 * SINGLE_TOL
    # linear XEB on the partial-slice amplitudes (analytics.py:46-58)
    n = 53
    f_ours = O.xeb(probs, n)
    f_ref = (2.0 ** n / probs.size) * float(g["amps_probsum"]) - 1.0
    assert measured(abs(f_ours - f_ref), 'xeb_abs') < 1e-3
    # bitstring indexing: row mask -> layout bitstring with s1 spliced
    assert len(tab.amplitudes) == 1 << len(tab.open_qubits)
    bs = tab.bitstring(1)
    assert bs[tab.open_qubits[-1]] == "1" and bs.count("1") == 1


def test_head_program_info(gpu, workloads):
    w = workloads("c4")
    prog = tnb.head_program(w.tn, w.tree, w.sliced, "single")
    assert prog.info.n_steps_tc >= 5
    assert abs(prog.info.flops_per_slice - 8.0 * w.tc_per_slice) / (8.0 * w.tc_per_slice) < 1e-12


@pytest.mark.parametrize("name,rng_", [("s8", (0, 16)), ("m12", (0, 4))])
def test_cross_slice_reuse_bit_identical(gpu, workloads, name, rng_):
    """TNB_FLAG_REUSE_SLICES skips steps whose mask bits did not change; the
    head vector must be bit-identical to full recomputation."""
    from paper_2103_03074_b200 import _lib, engine as E

    w = workloads(name)
    base = E.head_program(w.tn, w.tree, w.sliced, "single", flags=0)
    ref = base.run_range(*rng_)
    reuse = E.head_program(w.tn, w.tree, w.sliced, "single", flags=_lib.TNB_FLAG_REUSE_SLICES)
    reuse.set_timing(True)
    got = reuse.run_range(*rng_)
    assert np.array_equal(got, ref)
    assert reuse.timing()["steps_reused"] > 0
    # continuing with the next range reuses across calls, still bit-identical
    a, b = rng_
    assert np.array_equal(reuse.run_range(b, 2 * b - a), base.run_range(b, 2 * b - a))


@pytest.mark.parametrize("name", ["m12", "c2", "c3"])
def test_fused_staging_vs_staged(gpu, workloads, name):
    """Operands written by the producer GEMM's epilogue (default) and operands
    staged by the permute/split kernel (TNB_FLAG_NO_FUSE) both match the
    reference golden head slice; the fused program launches fewer kernels."""
    from paper_2103_03074_b200 import _lib, engine as E

    w = workloads(name)
    g = golden(name)
    stride = int(g["stride"])
    ref = g["head_single_0_1_sub"]
    fused = E.head_program(w.tn, w.tree, w.sliced, "single", flags=0)
    staged = E.head_program(w.tn, w.tree, w.sliced, "single", flags=_lib.TNB_FLAG_NO_FUSE)
    assert fused.info.n_steps_fused > 0 and staged.info.n_steps_fused == 0
    assert fused.info.kernels_per_slice < staged.info.kernels_per_slice
    hf = fused.run_range(0, 1)
    hs = staged.run_range(0, 1)
    ef, es = rel_l2(hf[::stride], ref), rel_l2(hs[::stride], ref)
    assert ef < SINGLE_TOL and es < SINGLE_TOL, (ef, es)
    # the bound-based fp16 scale keeps fp32-level accuracy
    assert ef < 10 * max(es, 1e-6), (ef, es)
    assert measured(rel_l2(hf, hs)) < SINGLE_TOL


def test_fused_staging_c4_plan(gpu, workloads):
    """C4: every tensor-core -> tensor-core edge is fused, most on the
    coalesced exchange path; no split-K producer is fused."""
    from paper_2103_03074_b200 import engine as E

    w = workloads("c4")
    prog = E.head_program(w.tn, w.tree, w.sliced, "single")
    assert prog.info.n_steps_fused >= 15
    # every large fused result takes a coalesced store path; the few on
    # per-element stores are small
    assert prog.info.n_steps_fused_fast >= prog.info.n_steps_fused - 8
