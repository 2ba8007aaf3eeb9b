"""Golden vectors for the analytics path, produced by the UNMODIFIED reference
(tncut.analytics) in the build container; committed so the GPU box (no
/root/reference) can check the device analytics against the reference."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from tncut import analytics as A  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "analytics", "golden.npz")
rng = np.random.default_rng(7)
n = 20
probs = A.porter_thomas_sample(n, 1 << 14, rng)
probs[:5] = 0.0  # zeros exercise the log-scale lower edge
rep = A.xeb(probs, n)
out = {"n": n, "probs": probs, "xeb": [rep.L, rep.f_xeb, rep.p_min, rep.p_max],
       "ks": A.ks_to_porter_thomas(probs, n), "mixed": A.mixed_xeb(probs, n, 1000)}
for scale in ("linear_Np", "log"):
    rows = A.histogram(probs, n, bins=40, scale=scale)
    out[f"hist_{scale}"] = np.array([[r.bin_lo, r.bin_hi, r.density, r.pt_density] for r in rows])
desc = np.sort(probs)[::-1].copy()
out["post"] = np.array(A.postselect_curve(desc, n, points=50))


class _T:  # the attributes marginal_and_conditional reads
    open_qubits = list(range(14))
    probabilities = probs


m, cond, f = A.marginal_and_conditional(_T())
out["marginal"] = [m, f]
out["cond_sub"] = cond[::97]
np.savez_compressed(OUT, **out)
print("wrote", OUT)
