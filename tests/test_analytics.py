"""Analytics: the numpy oracle pinned to the reference's
own outputs (CPU), and the device reductions of paper_2103_03074_b200.analytics
against both (GPU)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden


def _g():
    return golden("analytics")


def test_oracle_analytics_match_reference_goldens():
    from oracle import analytics_np as O

    g = _g()
    n, p = int(g["n"]), g["probs"]
    L, f, lo, hi = O.xeb(p, n)
    assert [L, f, lo, hi] == list(g["xeb"])
    assert O.ks_to_porter_thomas(p, n) == float(g["ks"])
    assert O.mixed_xeb(p, n, 1000) == float(g["mixed"])
    for scale in ("linear_Np", "log"):
        edges, dens, pt = O.histogram(p, n, bins=40, scale=scale)
        ref = g[f"hist_{scale}"]
        assert np.array_equal(edges[:-1], ref[:, 0]) and np.array_equal(edges[1:], ref[:, 1])
        assert np.array_equal(dens, ref[:, 2]) and np.array_equal(pt, ref[:, 3])
    post = O.postselect_curve(np.sort(p)[::-1], n, points=50)
    assert np.array_equal(np.array(post), g["post"])
    m, cond, fc = O.marginal_and_conditional(p, 14)
    assert [m, fc] == list(g["marginal"]) and np.array_equal(cond[::97], g["cond_sub"])


@pytest.mark.gpu
def test_device_analytics_match_reference(gpu):
    from paper_2103_03074_b200 import analytics as A

    g = _g()
    n, p = int(g["n"]), g["probs"]
    rep = A.xeb(p, n)
    L, f, lo, hi = g["xeb"]
    assert rep.L == L and rep.p_min == lo and rep.p_max == hi
    assert abs(rep.f_xeb - f) < 1e-12
    assert abs(A.ks_to_porter_thomas(p, n) - float(g["ks"])) < 1e-14
    assert abs(A.mixed_xeb(p, n, 1000) - float(g["mixed"])) < 1e-12
    for scale in ("linear_Np", "log"):
        rows = A.histogram(p, n, bins=40, scale=scale)
        got = np.array([[r.bin_lo, r.bin_hi, r.density, r.pt_density] for r in rows])
        assert np.array_equal(got, g[f"hist_{scale}"]), scale  # edges exact, counts exact
    post = A.postselect_curve(np.sort(p)[::-1].copy(), n, points=50)
    ref = g["post"]
    assert np.array_equal(np.array(post)[:, 0], ref[:, 0])
    assert np.max(np.abs(np.array(post)[:, 1] - ref[:, 1])) < 1e-12

    class T:
        open_qubits = list(range(14))
        probabilities = p
        amplitudes = np.sqrt(p)

    m, cond, fc = A.marginal_and_conditional(T())
    assert abs(m - g["marginal"][0]) < 1e-15 * 2 ** 14 and abs(fc - g["marginal"][1]) < 1e-12
    assert np.allclose(cond[::97], g["cond_sub"], rtol=1e-14, atol=0)


@pytest.mark.gpu
def test_device_analytics_errors_and_device_sort(gpu):
    import torch

    from paper_2103_03074_b200 import analytics as A

    with pytest.raises(A.EmptyInput):
        A.xeb(np.array([]), 10)
    with pytest.raises(A.NotSorted):
        A.postselect_curve(np.array([0.1, 0.3, 0.2]), 3)
    with pytest.raises(ValueError):
        A.histogram(np.array([0.1]), 3, bins=0)
    with pytest.raises(A.ZeroMarginal):
        class Z:
            open_qubits = [0, 1]
            probabilities = np.zeros(4)
            amplitudes = np.zeros(4)
        A.marginal_and_conditional(Z())
    with pytest.raises(A.IncompleteEnumeration):
        class I:
            open_qubits = [0, 1]
            probabilities = np.ones(3)
            amplitudes = np.ones(3)
        A.marginal_and_conditional(I())
    rng = np.random.default_rng(3)
    p = rng.exponential(size=100_003)
    t = A.sort_desc(torch.from_numpy(p).cuda())
    assert np.array_equal(t.cpu().numpy(), np.sort(p)[::-1])


@pytest.mark.gpu
def test_device_analytics_on_tail_amplitudes(gpu, workloads):
    """Amplitudes that never leave HBM: tail program output -> device XEB."""
    import torch

    from oracle import analytics_np as O
    from paper_2103_03074_b200 import analytics as A, engine as E

    w = workloads("m12")
    tn, tree = w.tn, w.tree
    hv = E.compute_head_vector(tn, tree, w.sliced, None, slice_range=(0, 2), precision="single")
    tab = E.tail_amplitudes_unchecked(tn, tree, hv, precision="single")
    amps = torch.from_numpy(np.asarray(tab.amplitudes)).cuda()
    rep = A.xeb(amps, 53)
    a64 = np.asarray(tab.amplitudes).astype(np.complex128)
    p64 = a64.real ** 2 + a64.imag ** 2  # the device's |a|^2 (fp64, no hypot)
    L, f, lo, hi = O.xeb(p64, 53)
    assert rep.L == L and abs(rep.f_xeb - f) <= 1e-12 * max(1.0, abs(f))
    assert rep.p_max == hi and rep.p_min == lo
    assert abs(A.ks_to_porter_thomas(amps, 53) - O.ks_to_porter_thomas(p64, 53)) < 1e-12
