"""Known-answer vectors at the BASELINE configs' real slice ranges (run HERE).

Round-1 goldens pinned one slice per Sycamore-scale config.  This script
drives the unmodified reference engine over the ranges SURVEY 8(d) names
and over non-default s1 (the batched-s1 path), and writes
``tests/golden/<name>/golden_ranges.npz``:

* ``c2``:  ``compute_head_vector(slice_range=(0, 8), precision="single",
  mode="fixed")`` (engine.py:242-310) stored in FULL (2^11), the blocked
  reference tail ``compute_tail_amplitudes`` (engine.py:313-378) in full
  (2^10), the reference ``analytics.xeb`` (analytics.py:46-58) of those
  amplitudes at n=53 and the conditional XEB (analytics.py:159-177);
  plus the 4 assignments of the two lowest closed qubits (s1 != 0,
  network.py:65-77) on slice 0, head + amplitudes in full.
* ``m12``: the 8 assignments of the three lowest closed qubits, slices
  [0, 2) -- the range ``tests/test_batched.py`` batches -- head (stride 64
  + norm) and the head-absorbed tail (reference greedy_order +
  contract_tree, as make_goldens.py).
* ``c4``:  slices [0, 4) in fixed AND free mode (engine.py:292-298),
  head stride 64 + norm; amplitudes of the fixed sum (absorbed tail),
  stride 16 + norm + both XEBs on the full vector.
* ``c3``:  slices [0, 4), fixed; head stride 4, amplitudes stride 16,
  XEBs.

Usage: ``python tests/golden/make_range_goldens.py m12 c2 c4 c3``.
"""

from __future__ import annotations

import dataclasses
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_goldens import absorbed_tail, load, sub  # noqa: E402  (inserts the reference path)
from tncut import analytics as tanalytics  # noqa: E402
from tncut import engine as tengine  # noqa: E402


def xebs(amps, n2):
    probs = np.abs(np.asarray(amps, dtype=np.complex128)) ** 2
    f53 = tanalytics.xeb(probs, 53).f_xeb
    cond = probs / probs.sum()
    fc = tanalytics.xeb(cond, n2).f_xeb
    return np.array([f53, fc])


def s1_variants(tn, nq):
    closed = sorted(tn.fixed_output_bits)
    out = []
    for v in range(1 << nq):
        s = dict(tn.fixed_output_bits)
        for i, q in enumerate(closed[:nq]):
            s[q] = (v >> (nq - 1 - i)) & 1
        out.append("".join(str(s[q]) for q in closed))
    return out


def head(tn, tree, sliced, s1, a, b, mode, name):
    st = tengine.EngineStats()
    t0 = time.time()
    hv = tengine.compute_head_vector(tn, tree, sliced, s1, slice_range=(a, b),
                                     precision="single", mode=mode, stats=st)
    dt = time.time() - t0
    print(f"[{name}] head s1={s1 if s1 is None else s1[:8] + '..'} [{a},{b}) {mode}: "
          f"{dt:.1f}s", flush=True)
    return hv, st, dt


def make(name):
    c, tn, tree, doc = load(name)
    sliced = doc["slices"]
    n_e = len(sliced)
    n2 = len(doc["open_qubits"])
    _, _, _, _, cut = tengine._split(tn, tree)
    out = {}
    t_all = time.time()
    if name == "c2":
        hv, st, dt = head(tn, tree, sliced, None, 0, 8, "fixed", name)
        out["head_fixed_0_8"] = hv.data
        out["head_fixed_0_8_stats"] = np.array([st.multiplications, st.head_contractions, 0,
                                                st.steps_executed])
        out["head_fixed_0_8_cpu_s"] = np.array(dt)
        full = dataclasses.replace(hv, slice_range=(0, 1 << n_e))
        amps = tengine.compute_tail_amplitudes(tn, tree, full, precision="single").amplitudes
        out["amps_fixed_0_8"] = amps
        out["xeb_fixed_0_8"] = xebs(amps, n2)
        s1s = s1_variants(tn, 2)
        out["s1_list"] = np.array(s1s)
        for i, s1 in enumerate(s1s):
            hv, _, _ = head(tn, tree, sliced, s1, 0, 1, "fixed", name)
            out[f"s1_{i}_head_0_1"] = hv.data
            out[f"s1_{i}_provenance"] = np.array(hv.provenance)
            full = dataclasses.replace(hv, slice_range=(0, 1 << n_e))
            out[f"s1_{i}_amps_0_1"] = tengine.compute_tail_amplitudes(
                tn, tree, full, precision="single").amplitudes
    elif name == "m12":
        stride, amp_stride = 64, 256
        s1s = s1_variants(tn, 3)
        out["s1_list"] = np.array(s1s)
        out["stride"] = np.array(stride)
        out["amps_stride"] = np.array(amp_stride)
        for i, s1 in enumerate(s1s):
            hv, _, _ = head(tn, tree, sliced, s1, 0, 2, "fixed", name)
            out[f"s1_{i}_head_0_2_sub"], out[f"s1_{i}_head_0_2_norm2"] = sub(hv.data, stride)
            out[f"s1_{i}_provenance"] = np.array(hv.provenance)
            tn_s = tn.repin(tengine.normalize_s1(tn, s1))
            amps = absorbed_tail(tn_s, tree, hv.data, sorted(cut), np.complex128)
            out[f"s1_{i}_amps_0_2_sub"], out[f"s1_{i}_amps_0_2_norm2"] = sub(amps, amp_stride)
    elif name in ("c4", "c3"):
        stride, amp_stride = (64, 16) if name == "c4" else (4, 16)
        out["stride"] = np.array(stride)
        out["amps_stride"] = np.array(amp_stride)
        modes = ("fixed", "free") if name == "c4" else ("fixed",)
        for mode in modes:
            hv, st, dt = head(tn, tree, sliced, None, 0, 4, mode, name)
            key = f"head_{mode}_0_4"
            out[key + "_sub"], out[key + "_norm2"] = sub(hv.data, stride)
            out[key + "_stats"] = np.array([st.multiplications, st.head_contractions, 0,
                                            st.steps_executed])
            out[key + "_cpu_s"] = np.array(dt)
            out[key + "_provenance"] = np.array(hv.provenance)
            if mode == "fixed":
                t0 = time.time()
                amps = absorbed_tail(tn, tree, hv.data, sorted(cut), np.complex128)
                print(f"[{name}] absorbed tail {time.time() - t0:.1f}s", flush=True)
                out["amps_fixed_0_4_sub"], out["amps_fixed_0_4_norm2"] = sub(amps, amp_stride)
                out["xeb_fixed_0_4"] = xebs(amps, n2)
    else:
        raise SystemExit(f"unknown config {name}")
    np.savez_compressed(os.path.join(HERE, name, "golden_ranges.npz"), **out)
    print(f"[{name}] range goldens in {time.time() - t_all:.1f}s", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        make(n)
