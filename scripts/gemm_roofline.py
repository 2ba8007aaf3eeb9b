"""Per-launch roofline of the tcgen05 GEMMs of one contraction.

    python scripts/gemm_roofline.py DEBUG_LOG NCU_CSV [n_slices]

DEBUG_LOG: stderr of a run with TNB_DEBUG_GEMM=1 (plan-time shapes, one
line per tensor-core step, plan order, with its hoisted flag).  NCU_CSV:
``ncu --csv -k regex:"gemm_(f16x3|skinny)" --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,
sm__cycles_elapsed.avg.per_second`` of the same run (guard re-runs off:
TNB_SCALE_GUARD_BITS=-1, so launches map 1:1 to steps: hoisted steps once,
then the per-slice steps for every slice).

Per launch: algorithmic complex FLOP (8 M N K = 2 M Np Kp), tensor-pipe
busy (ncu), DRAM bytes and GB/s against the measured HBM peak, the bound
(tensor or HBM: whichever fraction is larger) and the wave efficiency of
the persistent grid (work units / (waves x CTA units)).  The summary is
time-weighted: sum(t * max(tensor, hbm)) / sum(t) = the fraction of their
own roofline the GEMMs run at."""
import collections
import csv
import io
import json
import math
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6450.0


def steps(log):
    pat = re.compile(r"TNB_GEMM step (\d+) M (\d+) Np (\d+) Kp (\d+) cg (\d+) nb (\d+) splits (\d+) "
                     r"fused_out (\d+) rows_fused (\d+) cols_fused (\d+) hoisted (\d+) grid (\d+)(?: skinny (\d+))?")
    out = []
    for line in open(log):
        m = pat.search(line)
        if m:
            v = [int(x) if x is not None else 0 for x in m.groups()]
            out.append(dict(step=v[0], M=v[1], Np=v[2], Kp=v[3], cg=v[4], nb=v[5], splits=v[6],
                            fused=v[7], hoisted=v[10], grid=v[11], skinny=v[12]))
    return out


def launches(path):
    txt = open(path).read().split("\n")
    start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    by = collections.OrderedDict()
    for r in rows:
        d = by.setdefault(r["ID"], {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                  "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}[unit]
        byte_units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                      "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        if unit in byte_units:
            v *= byte_units[unit]
        d[r["Metric Name"]] = v
    return list(by.values())


def main():
    st = steps(sys.argv[1])
    ln = launches(sys.argv[2])
    n_sl = int(sys.argv[3]) if len(sys.argv) > 3 else None
    order = [s for s in st if s["hoisted"]]
    per = [s for s in st if not s["hoisted"]]
    if n_sl is None:
        n_sl = max(1, (len(ln) - len(order)) // max(1, len(per)))
    order += per * n_sl
    if len(order) != len(ln):
        print(f"warning: {len(ln)} launches vs {len(order)} planned GEMMs; matching the first "
              f"{min(len(ln), len(order))}", file=sys.stderr)
    peak = hbm_peak()
    units = 148
    tot_t = tot_w = tot_f = 0.0
    agg = {"tensor": [0.0, 0.0], "hbm": [0.0, 0.0]}
    print(f"{'step':>5} {'M':>7} {'N':>7} {'K':>7} {'nb':>3} {'sp':>2} {'ms':>8} {'TF/s':>6} "
          f"{'tens%':>6} {'GB':>6} {'GB/s':>6} {'hbm%':>5} {'wave%':>5} bound")
    for s, l in zip(order, ln):
        t = l["gpu__time_duration.sum"]
        fl = 2.0 * s["M"] * s["Np"] * s["Kp"]
        by = l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
        tens = l.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) / 100
        hbm = by / t / 1e9 / peak
        tiles = math.ceil(s["M"] / (128 * s["cg"])) * math.ceil(s["Np"] / s["nb"]) * s["splits"]
        u = units // s["cg"]
        wave = tiles / (math.ceil(tiles / u) * u)
        frac = max(tens, hbm)
        bound = "tensor" if tens >= hbm else "hbm"
        if s.get("skinny"):
            bound = "hbm*"  # FP32-pipe skinny kernel: judged against HBM
        agg[bound.rstrip("*")][0] += t
        agg[bound.rstrip("*")][1] += t * (hbm if s.get("skinny") else frac)
        tot_t += t
        tot_w += t * (hbm if s.get("skinny") else frac)
        tot_f += fl
        print(f"{s['step']:5d} {s['M']:7d} {s['Np'] // 2:7d} {s['Kp'] // 2:7d} {s['nb']:3d} {s['splits']:2d} "
              f"{t * 1e3:8.3f} {fl / t / 1e12:6.1f} {100 * tens:6.1f} {by / 1e9:6.2f} {by / t / 1e9:6.0f} "
              f"{100 * hbm:5.1f} {100 * wave:5.1f} {bound}")
    print(f"\nGEMMs {len(ln)}: {tot_t * 1e3:.2f} ms, {tot_f / tot_t / 1e12:.1f} TFLOP/s algorithmic (ncu serialised, cold L2)")
    print(f"time-weighted fraction of own roofline max(tensor busy, DRAM/{peak:.0f} GB/s): {tot_w / tot_t:.3f}")
    for b, (t, w) in agg.items():
        if t:
            print(f"  {b}-bound launches: {t * 1e3:.2f} ms ({100 * t / tot_t:.1f}%), at {w / t:.3f} of their bound")


if __name__ == "__main__":
    main()
