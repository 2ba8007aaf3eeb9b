"""GPU parity at the BASELINE configs' real slice ranges and at non-default
s1, against goldens from the UNMODIFIED reference engine
(tests/golden/make_range_goldens.py -> golden_ranges.npz):

* m12: 8 closed-bit assignments (s1 != 0 for 7 of them), slices [0, 2):
  per-s1 calls, the same calls from 8 concurrent threads (the reference's
  ``cli run --threads`` fan-out, cli.py:367-380), and ONE batched-s1
  contraction (batched.py) -- heads and head-absorbed amplitudes;
* c2: [0, 8) fixed, full head and full amplitudes + XEBs; 4 s1 on slice 0;
* c4: [0, 4) fixed AND free; amplitudes + XEBs of the fixed sum;
* c3: [0, 4) fixed.

Every comparison prints its measured error (run pytest with -s or -rA to
see them).  Tolerances: 1e-4 relative L2 on head vectors and amplitudes,
1e-3 absolute on XEB (north_star); indices and bit order are exact by
construction (same positions compared).
"""

from __future__ import annotations

import os
import threading

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from conftest import GOLDEN, parity_report, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-4
XEB_TOL = 1e-3


def ranges_golden(name):
    path = os.path.join(GOLDEN, name, "golden_ranges.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_range_goldens.py {name}")
    return np.load(path)


report = parity_report


def check_sub(tag, ours, g, key, stride):
    """rel L2 on the stored subsample + relative error of the exact norm^2."""
    ours = np.asarray(ours).reshape(-1)
    e = rel_l2(ours[::stride], g[key + "_sub"])
    n2 = float(np.vdot(ours.astype(np.complex128), ours.astype(np.complex128)).real)
    en = abs(n2 / float(g[key + "_norm2"]) - 1.0)
    report(tag, rel_l2_sub=e, norm2_rel=en)
    assert e < TOL and en < 2 * TOL, tag
    return e


def xebs(amps, n2):
    from oracle import engine_np as O

    probs = np.abs(np.asarray(amps, dtype=np.complex128)) ** 2
    return O.xeb(probs, 53), O.xeb(probs / probs.sum(), n2)


# ---------------------------------------------------------------------------
# m12: non-default s1 (per call, threaded, batched)

def _m12_call(w, s1):
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s1, slice_range=(0, 2), precision="single")
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    return hv, tab


def test_m12_nondefault_s1_heads_and_amplitudes(gpu, workloads):
    w = workloads("m12")
    g = ranges_golden("m12")
    s1s = [str(s) for s in g["s1_list"]]
    stride, astride = int(g["stride"]), int(g["amps_stride"])
    assert len(set(s1s)) == 8
    for i, s1 in enumerate(s1s):
        hv, tab = _m12_call(w, s1)
        assert hv.provenance == str(g[f"s1_{i}_provenance"])  # reference hash, same s1
        check_sub(f"m12 s1#{i} head [0,2)", hv.data, g, f"s1_{i}_head_0_2", stride)
        check_sub(f"m12 s1#{i} amplitudes", tab.amplitudes, g, f"s1_{i}_amps_0_2", astride)


def test_m12_concurrent_threads_mixed_s1(gpu, workloads):
    """8 threads, 8 different s1, same cached program: each result equals the
    reference's for ITS s1 (upload+run is one critical section)."""
    w = workloads("m12")
    g = ranges_golden("m12")
    s1s = [str(s) for s in g["s1_list"]]
    stride, astride = int(g["stride"]), int(g["amps_stride"])
    results = [None] * len(s1s)
    errors = []
    barrier = threading.Barrier(len(s1s))

    def work(i):
        try:
            barrier.wait()
            for _ in range(2):  # twice, so uploads of other s1 interleave
                results[i] = _m12_call(w, s1s[i])
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(s1s))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i, (hv, tab) in enumerate(results):
        assert hv.provenance == str(g[f"s1_{i}_provenance"])
        check_sub(f"m12 threaded s1#{i} head", hv.data, g, f"s1_{i}_head_0_2", stride)
        check_sub(f"m12 threaded s1#{i} amplitudes", tab.amplitudes, g, f"s1_{i}_amps_0_2", astride)


def test_m12_batched_s1_against_reference(gpu, workloads):
    """ONE contraction with the three closed qubits' legs open gives all 8
    head vectors; each equals the reference's per-s1 head."""
    from paper_2103_03074_b200.batched import compute_head_vectors_batched

    w = workloads("m12")
    g = ranges_golden("m12")
    s1s = [str(s) for s in g["s1_list"]]
    stride, astride = int(g["stride"]), int(g["amps_stride"])
    hvs = compute_head_vectors_batched(w.tn, w.tree, w.sliced, s1s, slice_range=(0, 2),
                                       precision="single")
    for i, hv in enumerate(hvs):
        assert hv.provenance == str(g[f"s1_{i}_provenance"])
        check_sub(f"m12 batched s1#{i} head", hv.data, g, f"s1_{i}_head_0_2", stride)
        tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
        check_sub(f"m12 batched s1#{i} amplitudes", tab.amplitudes, g, f"s1_{i}_amps_0_2", astride)


# ---------------------------------------------------------------------------
# c2: [0, 8) in full, 4 s1

def test_c2_slices_0_8_full_vector(gpu, workloads):
    w = workloads("c2")
    g = ranges_golden("c2")
    st = tnb.EngineStats()
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 8),
                                 precision="single", stats=st)
    e = rel_l2(hv.data, g["head_fixed_0_8"])
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    ea = rel_l2(tab.amplitudes, g["amps_fixed_0_8"])
    f53, fc = xebs(tab.amplitudes, len(tab.open_qubits))
    gx = g["xeb_fixed_0_8"]
    report("c2 [0,8) full", head_rel_l2=e, amps_rel_l2=ea, xeb53_abs=abs(f53 - gx[0]),
           xeb_cond_abs=abs(fc - gx[1]))
    assert e < TOL and ea < TOL
    assert abs(f53 - gx[0]) < XEB_TOL and abs(fc - gx[1]) < XEB_TOL
    assert [st.multiplications, st.head_contractions, st.steps_executed] == \
        [int(g["head_fixed_0_8_stats"][0]), int(g["head_fixed_0_8_stats"][1]),
         int(g["head_fixed_0_8_stats"][3])]


def test_c2_nondefault_s1_single_and_batched(gpu, workloads):
    from paper_2103_03074_b200.batched import compute_head_vectors_batched

    w = workloads("c2")
    g = ranges_golden("c2")
    s1s = [str(s) for s in g["s1_list"]]
    hvs_b = compute_head_vectors_batched(w.tn, w.tree, w.sliced, s1s, slice_range=(0, 1),
                                         precision="single")
    for i, s1 in enumerate(s1s):
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s1, slice_range=(0, 1),
                                     precision="single")
        assert hv.provenance == str(g[f"s1_{i}_provenance"])
        tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
        tab_b = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hvs_b[i], precision="single")
        e, ea = rel_l2(hv.data, g[f"s1_{i}_head_0_1"]), rel_l2(tab.amplitudes, g[f"s1_{i}_amps_0_1"])
        eb = rel_l2(hvs_b[i].data, g[f"s1_{i}_head_0_1"])
        eba = rel_l2(tab_b.amplitudes, g[f"s1_{i}_amps_0_1"])
        report(f"c2 s1#{i} slice 0", head=e, amps=ea, batched_head=eb, batched_amps=eba)
        assert max(e, ea, eb, eba) < TOL


# ---------------------------------------------------------------------------
# c4 / c3: the bench configs' ranges

def test_c4_slices_0_4_fixed_and_free(gpu, workloads):
    w = workloads("c4")
    g = ranges_golden("c4")
    stride, astride = int(g["stride"]), int(g["amps_stride"])
    for mode in ("fixed", "free"):
        st = tnb.EngineStats()
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 4),
                                     precision="single", mode=mode, stats=st)
        key = f"head_{mode}_0_4"
        assert hv.provenance == str(g[key + "_provenance"])
        check_sub(f"c4 [0,4) {mode} head", hv.data, g, key, stride)
        assert [st.multiplications, st.head_contractions] == [int(g[key + "_stats"][0]),
                                                              int(g[key + "_stats"][1])]
        if mode == "fixed":
            tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
            check_sub("c4 [0,4) fixed amplitudes", tab.amplitudes, g, "amps_fixed_0_4", astride)
            f53, fc = xebs(tab.amplitudes, len(tab.open_qubits))
            gx = g["xeb_fixed_0_4"]
            report("c4 [0,4) XEB", xeb53_abs=abs(f53 - gx[0]), xeb_cond_abs=abs(fc - gx[1]))
            assert abs(f53 - gx[0]) < XEB_TOL and abs(fc - gx[1]) < XEB_TOL


def test_c3_slices_0_4(gpu, workloads):
    w = workloads("c3")
    g = ranges_golden("c3")
    stride, astride = int(g["stride"]), int(g["amps_stride"])
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 4),
                                 precision="single")
    assert hv.provenance == str(g["head_fixed_0_4_provenance"])
    check_sub("c3 [0,4) head", hv.data, g, "head_fixed_0_4", stride)
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    check_sub("c3 [0,4) amplitudes", tab.amplitudes, g, "amps_fixed_0_4", astride)
    f53, fc = xebs(tab.amplitudes, len(tab.open_qubits))
    gx = g["xeb_fixed_0_4"]
    report("c3 [0,4) XEB", xeb53_abs=abs(f53 - gx[0]), xeb_cond_abs=abs(fc - gx[1]))
    assert abs(f53 - gx[0]) < XEB_TOL and abs(fc - gx[1]) < XEB_TOL
