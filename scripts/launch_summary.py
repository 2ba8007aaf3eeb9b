"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under `| head`

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
seq = []
for r in data:
    ms = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].split("(")[0].replace("tnb::<unnamed>::", "").replace("void ", "")[:48]
    agg[name][0] += 1
    agg[name][1] += ms
    tot += ms
    seq.append((name, ms))
print(f"launches {len(data)}  total {tot:.2f} ms (ncu: serialised, cold L2)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:48s} {n:5d} {t:9.2f} ms {100 * t / tot:5.1f}%")
if len(sys.argv) > 2:
    top = sorted(seq, key=lambda x: -x[1])[: int(sys.argv[2])]
    for name, ms in top:
        print(f"    {name:48s} {ms:8.3f} ms")
