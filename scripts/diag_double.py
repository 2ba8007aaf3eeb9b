"""Time one head slice in double precision (the reference's default,
engine.py:248) on the fp64 path and compare it with the single-precision
head of the same slice:  python scripts/diag_double.py c4 [slices]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import engine as E  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = tnb.load_workload(name)
for prec in ("double", "single"):
    prog = E.head_program(w.tn, w.tree, w.sliced, prec, device=0)
    prog.set_timing(1)
    prog.run_range(0, n, "fixed")  # warm
    t0 = time.time()
    out = prog.run_range(0, n, "fixed")
    wall = time.time() - t0
    t = prog.timing()
    flops = 8.0 * w.tc_per_slice * n
    print(prec, {k: round(v, 2) if isinstance(v, float) else v for k, v in t.items()},
          f"wall {wall:.2f}s  {flops / (t['total_ms'] / 1e3) / 1e12:.2f} TFLOP/s", flush=True)
    if prec == "double":
        dbl = out
    else:
        print("single vs double rel L2", float(np.linalg.norm(out - dbl) / np.linalg.norm(dbl)))
    del prog
    E.clear_cache()
