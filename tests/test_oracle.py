"""Pin the numpy oracle against the reference's own known answers (CPU).

Golden vectors come from the unmodified reference engine and state-vector
simulator (tests/golden/make_goldens.py).  The oracle restates the same
numpy operations, so on identical inputs it must agree bit-for-bit.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import engine_np as O


def test_c1_head_full_range_bit_exact(workloads):
    w = workloads("c1")
    g = golden("c1")
    h = O.head_vector(w.tn, w.tree, w.sliced, precision="double")
    assert np.array_equal(h, g["head_full_double"])
    hs = O.head_vector(w.tn, w.tree, w.sliced, precision="single")
    assert np.array_equal(hs, g["head_full_single"])


@pytest.mark.parametrize("rng_", [(0, 8), (8, 16), (0, 4), (4, 8), (3, 11)])
@pytest.mark.parametrize("mode", ["fixed", "free"])
def test_c1_ranges_and_modes_bit_exact(workloads, rng_, mode):
    w = workloads("c1")
    g = golden("c1")
    p = O.head_vector(w.tn, w.tree, w.sliced, rng_, "double", mode)
    assert np.array_equal(p, g[f"head_{mode}_{rng_[0]}_{rng_[1]}"])


def test_c1_fixed_partials_compose(workloads):
    w = workloads("c1")
    g = golden("c1")
    parts = [((0, 8), g["head_fixed_0_8"]), ((8, 16), g["head_fixed_8_16"])]
    assert np.array_equal(O.combine_partials(parts), g["head_full_double"])


def test_c1_tail_blocked_and_absorbed(workloads):
    w = workloads("c1")
    g = golden("c1")
    h = g["head_full_double"]
    blocked = O.tail_blocked(w.tn, w.tree, h, space_cap=8, precision="double")
    assert np.array_equal(blocked, g["amps_engine"][0])
    absorbed = O.tail_absorbed(w.tn, w.tree, h, precision="double")
    assert np.abs(absorbed - g["amps_statevector"][0]).max() < 1e-12
    st = O.Stats()
    O.tail_blocked(w.tn, w.tree, h, space_cap=6, precision="double", stats=st)
    assert [st.multiplications, st.tail_contractions, st.steps_executed] == \
        [int(g["tail_stats_cap6"][0]), int(g["tail_stats_cap6"][2]), int(g["tail_stats_cap6"][3])]


def test_c1_all_amplitudes_vs_statevector(workloads):
    """All 2^12 amplitudes: 256 closed-bit repins x 16 open amplitudes."""
    w = workloads("c1")
    g = golden("c1")
    closed = sorted(w.tn.fixed_output_bits)
    for s1v in range(0, 256, 17):
        bits = {q: (s1v >> (len(closed) - 1 - i)) & 1 for i, q in enumerate(closed)}
        tn = w.tn.repin(bits)
        h = O.head_vector(tn, w.tree, w.sliced, precision="double")
        a = O.tail_blocked(tn, w.tree, h, space_cap=8, precision="double")
        assert np.array_equal(a, g["amps_engine"][s1v])
        assert np.abs(a - g["amps_statevector"][s1v]).max() < 1e-12


def test_c1_stats(workloads):
    w = workloads("c1")
    g = golden("c1")
    st = O.Stats()
    O.head_vector(w.tn, w.tree, w.sliced, precision="double", stats=st)
    assert [st.multiplications, st.head_contractions, st.steps_executed] == \
        [int(g["head_stats"][0]), int(g["head_stats"][1]), int(g["head_stats"][3])]


def test_c1_contract_tree(workloads):
    w = workloads("c1")
    g = golden("c1")
    asg = {ix: (5 >> (w.n_e - 1 - p)) & 1 for p, ix in enumerate(w.sliced)}
    assert np.array_equal(O.contract_tree(w.tn, w.tree, asg), g["contract_tree_mask5"])


@pytest.mark.parametrize("rng_", [(0, 4), (0, 1), (4, 8)])
def test_s8_head_single_bit_exact(workloads, rng_):
    w = workloads("s8")
    g = golden("s8")
    stride = int(g["stride"])
    p = O.head_vector(w.tn, w.tree, w.sliced, rng_, "single")
    a, b = rng_
    assert np.array_equal(p[::stride], g[f"head_single_{a}_{b}_sub"])
    assert abs(float(np.vdot(p, p).real) / float(g[f"head_single_{a}_{b}_norm2"]) - 1) < 1e-6


def test_s8_tail_formulations_agree(workloads):
    w = workloads("s8")
    g = golden("s8")
    p = O.head_vector(w.tn, w.tree, w.sliced, (0, 4), "single")
    a = O.tail_absorbed(w.tn, w.tree, p.astype(np.complex128), precision="double")
    assert rel_l2(a, g["amps_sub"]) < 1e-5          # vs reference blocked tail (single)
    assert rel_l2(a, g["amps_absorbed"]) < 1e-12    # vs reference greedy+contract_tree


@pytest.mark.parametrize("name,nslices", [("m12", 1), ("c2", 1), ("c3", 1), ("c4", 1),
                                          ("c5_26", 2)])
def test_large_config_goldens_consistent(workloads, name, nslices):
    """The big-config goldens exist and carry the reference's stats contract:
    multiplications per slice == the order file's per-subtask tc."""
    w = workloads(name)
    g = golden(name)
    st = g[f"head_single_0_{nslices}_stats"]
    assert int(st[0]) == nslices * w.tc_per_slice
    assert int(st[1]) == nslices


def test_sweep_plans_match_survey(workloads):
    """C5: the C4 tree re-sliced at t = 26/28/30/32 gives n_e 63/58/53/48."""
    assert [workloads(n).n_e for n in ("c5_26", "c5_28", "c4", "c5_32")] == [63, 58, 53, 48]
