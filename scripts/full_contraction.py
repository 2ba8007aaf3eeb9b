"""Complete head sum (ALL slices) of a co-optimised plan on one GPU, then the
tail amplitudes and their XEB -- the finished answer of a BASELINE config,
not a slice subset:
    python scripts/full_contraction.py c3_opt_b200 [batch_log2]
Prints one JSON line; consistency: the first 2^10 slices are also summed
by the per-slice path and compared."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_03074_b200 as tnb  # noqa: E402
from paper_2103_03074_b200 import analytics  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_opt_b200"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = tnb.load_workload(name)
total = 1 << w.n_e
chunk = min(total, 1 << 12)
# consistency: batched vs per-slice on the first chunk
a = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, min(chunk, 1 << 10)),
                            precision="single")
tnb.set_slice_batch(k)
b = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, min(chunk, 1 << 10)),
                            precision="single")
den = float(np.linalg.norm(a.data))
consistency = float(np.linalg.norm(a.data.astype(np.complex128) - b.data) / den)
tnb.clear_cache()
t0 = time.perf_counter()
parts = []
for lo in range(0, total, chunk):
    parts.append(tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(lo, lo + chunk),
                                         precision="single"))
head = tnb.reduce_partials(parts)  # aligned power-of-two partials: the fixed-mode tree
t1 = time.perf_counter()
tnb.set_slice_batch(0)
tab = tnb.compute_tail_amplitudes(w.tn, w.tree, head, precision="single")
t2 = time.perf_counter()
probs = np.abs(tab.amplitudes.astype(np.complex128)) ** 2
os.makedirs("gpurun_out", exist_ok=True)
np.save(os.path.join("gpurun_out", f"full_amps_{name}.npy"), tab.amplitudes)
x = analytics.xeb(probs, 53)
print(json.dumps({"plan": name, "n_e": w.n_e, "slices": total, "batch_log2": k,
                  "head_seconds": t1 - t0, "tail_seconds": t2 - t1,
                  "slices_per_s": total / (t1 - t0),
                  "flops_total": 8.0 * w.tc_per_slice * total,
                  "amplitudes": len(tab.amplitudes), "prob_sum": float(probs.sum()),
                  "xeb": x.f_xeb, "p_max": x.p_max, "consistency_batched_vs_per_slice": consistency,
                  "first_bitstrings": [tab.bitstring(i) for i in range(2)],
                  "first_amplitudes": [str(complex(v)) for v in tab.amplitudes[:2]]}), flush=True)
