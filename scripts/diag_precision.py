"""Single-precision error vs fp64 on one head slice range, per execution
path: SIMT fp32 only, tensor cores with staged operands, tensor cores with
fused staging (default).  Separates fp32-inherent error from the split-fp16
tensor-core arithmetic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import _lib, engine as E

def rel(a, b): return float(np.linalg.norm(np.asarray(a, complex) - b) / np.linalg.norm(b))
for name in sys.argv[1:] or ["m12", "c2"]:
    w = tnb.load_workload(name)
    d = E.head_program(w.tn, w.tree, w.sliced, "double").run_range(0, 2)
    out = []
    for label, flags in (("simt-fp32", _lib.TNB_FLAG_NO_TENSOR_CORES), ("tc-staged", _lib.TNB_FLAG_NO_FUSE), ("tc-fused", 0)):
        h = E.head_program(w.tn, w.tree, w.sliced, "single", flags=flags).run_range(0, 2)
        out.append(f"{label} {rel(h, d):.2e}")
        E.clear_cache()
    print(name, " | ".join(out), flush=True)
