"""Run one C4-family contraction for ncu / TNB_DEBUG_GEMM inspection:
    python scripts/diag_tree.py given c4 2        # reference tree, 2 slices
    python scripts/diag_tree.py reordered c4 16   # same slices, re-ordered tree
    python scripts/diag_tree.py batched c4 4      # 2^4 slices per contraction, 1 block
    python scripts/diag_tree.py plan c4_opt31_b200 1   # a frozen plan's own tree
One warm-up run first (compile + graphs), then the measured run; with
TNB_DIAG_SKIP_WARM=1 only the measured run (ncu -c counts stay small)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import engine as E  # noqa: E402
from paper_2103_03074_b200 import slice_batch as SB  # noqa: E402
from paper_2103_03074_b200.planner import cluster_small_steps  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "given"
name = sys.argv[2] if len(sys.argv) > 2 else "c4"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = tnb.load_workload(name)
if mode in ("given", "plan"):  # plan: any frozen workload's own tree, e.g. c4_opt31_b200
    prog = E.head_program(w.tn, w.tree, w.sliced, "single", device=0)
    rng = [(0, n), (n, 2 * n)]
elif mode == "reordered":
    wr = tnb.load_workload(name + "_reordered")
    hl, hs, _, _, cut = E._split(wr.tn, wr.tree)
    steps = cluster_small_steps({x: wr.tn.nodes[x].indices for x in hl}, hs, frozenset(wr.sliced))
    prog = E.get_program(E._leaf_entries(wr.tn, hl), E._steps_tuples(steps), list(wr.sliced),
                         sorted(cut), "single", 0)
    rng = [(0, n), (n, 2 * n)]
else:
    prog = SB.batched_program(w.tn, w.tree, w.sliced, n, "single", 0)
    rng = [(0, 1), (1, 2)]
prog.set_timing(int(os.environ.get("TNB_DIAG_TIMING", "2")))
reps = int(os.environ.get("TNB_DIAG_REPS", "1"))
rng = rng[:1] + rng[1:] * reps
if os.environ.get("TNB_DIAG_SKIP_WARM") == "1":
    rng = rng[1:]
for a, b in rng:
    prog.run_range(a, b, "fixed")
    t = prog.timing()
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}, flush=True)
