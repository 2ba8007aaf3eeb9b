import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200.batched import compute_head_vectors_batched
from test_batched import _s1_list
def rel(a, b): return float(np.linalg.norm(np.asarray(a, complex) - b) / np.linalg.norm(b))
for name, nq in (("c2", 3), ("m12", 2)):
    w = tnb.load_workload(name)
    closed = sorted(w.tn.fixed_output_bits)
    s1s = _s1_list(w.tn, closed[:nq])
    hvs = compute_head_vectors_batched(w.tn, w.tree, w.sliced, s1s, slice_range=(0, 2), precision="single")
    for s, hv in list(zip(s1s, hvs))[:3]:
        d = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s, slice_range=(0, 2), precision="double").data
        p = tnb.compute_head_vector(w.tn, w.tree, w.sliced, s, slice_range=(0, 2), precision="single").data
        print(name, s[:0] if False else "", "per-s1 vs fp64 %.2e  batched vs fp64 %.2e" % (rel(p, d), rel(hv.data, d)), flush=True)
