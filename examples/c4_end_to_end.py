"""End to end on the public API (what a user of the reference does):
plan -> head slices -> tail amplitudes -> XEB, on the frozen C4 workload.

    python examples/c4_end_to_end.py [--slices 64] [--plan given|reordered|batched] [--tsv amps.tsv]

* ``given``: the reference plan's tree as is (the bench headline path);
* ``reordered``: same slices, re-ordered head tree (``set_reorder``);
* ``batched``: same slices, 16 per contraction (``set_slice_batch(4)``).
All three return the same partial head vector for the same slice range.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import analytics  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", type=int, default=64)
    ap.add_argument("--plan", choices=["given", "reordered", "batched"], default="batched")
    ap.add_argument("--tsv", default=None, help="write the 2^20 rows as the reference's TSV")
    args = ap.parse_args()
    w = tnb.load_workload("c4")
    tnb.set_reorder(args.plan == "reordered")
    tnb.set_slice_batch(4 if args.plan == "batched" else 0)
    t0 = time.perf_counter()
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, args.slices),
                                 precision="single")
    t1 = time.perf_counter()
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    t2 = time.perf_counter()
    probs = np.abs(tab.amplitudes.astype(np.complex128)) ** 2
    print(f"plan={args.plan}: {args.slices} head slices in {t1 - t0:.2f} s "
          f"(incl. planning/compile on first use), tail {t2 - t1:.2f} s")
    print(f"head |v|^2 = {float(np.vdot(hv.data, hv.data).real):.6e}, "
          f"{len(tab.amplitudes)} amplitudes, first bitstring {tab.bitstring(0)}")
    print(f"linear XEB of this partial (a 2^-{w.n_e - int(np.log2(args.slices))} fraction of the "
          f"slice sum): {analytics.xeb(probs, 53).f_xeb:.6f}")
    if args.tsv:
        from paper_2103_03074_b200 import io

        t3 = time.perf_counter()
        io.write_amplitude_tsv(args.tsv, tab)  # byte-identical to tncut's writer
        print(f"{len(tab.amplitudes)} TSV rows in {time.perf_counter() - t3:.2f} s -> {args.tsv}")


if __name__ == "__main__":
    main()
