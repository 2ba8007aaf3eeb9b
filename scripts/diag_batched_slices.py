"""Per-class device time of batched-slice blocks (slice_batch.py):
    python scripts/diag_batched_slices.py c4 4 [blocks] [max_rank]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import slice_batch as SB  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 4
mr = int(sys.argv[4]) if len(sys.argv) > 4 else None
w = tnb.load_workload(name)
p = SB.batched_program(w.tn, w.tree, w.sliced, k, "single", 0, max_rank=mr)
p.set_timing(1)
for rep in range(3):
    p.run_range(rep * nb, (rep + 1) * nb, "fixed")
    t = p.timing()
    print({a: round(b, 3) if isinstance(b, float) else b for a, b in t.items()}, flush=True)
