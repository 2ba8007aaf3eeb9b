"""Host-side profile of the e2e bench step (public API, host buffers)."""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import engine as E  # noqa: E402

w = tnb.load_workload(sys.argv[1] if len(sys.argv) > 1 else "c4")
S = 2


def step(a):
    # as bench.py's e2e leg: every call's leaves arrive from the host
    prog = E.head_program(w.tn, w.tree, w.sliced, "single")
    prog._leaf_data = [None] * prog.n_leaves
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(a, a + S),
                                 precision="single")
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    return tab


for a in range(0, 3 * S, S):
    step(a)
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for a in range(10 * S, 13 * S, S):
    step(a)
pr.disable()
print(f"3 steps: {(time.perf_counter() - t0) * 1e3:.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
