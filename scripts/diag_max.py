"""Diagnostic: per-step output max vs the a-priori bound 2 K max|A| max|B|
(TNB_DEBUG_MAX), for the fp16-scale-from-bound design of fused staging."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TNB_DEBUG_MAX"] = "1"
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import engine

for name in sys.argv[1:]:
    w = tnb.load_workload(name)
    print("=== workload", name, file=sys.stderr, flush=True)
    prog = engine.head_program(w.tn, w.tree, w.sliced, "single")
    prog.run_range(0, 1, "fixed")
