"""Run a few head slices of a frozen plan (default c4_opt) once, for ncu /
TNB_DEBUG_FUSE inspection of its kernels:
    TNB_DEBUG_FUSE=1 python scripts/diag_plan_kernels.py c4_opt 2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import engine as E  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_opt"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = tnb.load_workload(name)
prog = E.head_program(w.tn, w.tree, w.sliced, "single", device=0)
prog.set_timing(1)
for s in range(n):
    prog.run_range(s, s + 1, "fixed")
    t = prog.timing()
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}, flush=True)
torch.cuda.synchronize()
