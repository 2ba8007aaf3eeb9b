"""numpy restatement of the reference analytics -- TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/tncut/analytics.py (line cites per function);
the checker for paper_2103_03074_b200.analytics (device reductions).  Pinned
against the reference's own outputs in tests/golden/analytics (CPU test).
"""

from __future__ import annotations

import math

import numpy as np


def xeb(probs, n):
    """analytics.py:46-58 -> (L, f_xeb, p_min, p_max)."""
    p = np.asarray(probs, dtype=np.float64).ravel()
    return p.size, (2.0 ** n / p.size) * float(p.sum()) - 1.0, float(p.min()), float(p.max())


def ks_to_porter_thomas(probs, n):
    """analytics.py:70-79: sup-distance of the empirical CDF of 2^n p (both
    step sides) to 1 - exp(-x)."""
    x = np.sort(np.asarray(probs, dtype=np.float64).ravel()) * 2.0 ** n
    L = x.size
    cdf = 1.0 - np.exp(-x)
    upper = np.arange(1, L + 1) / L
    return float(np.maximum(np.abs(upper - cdf), np.abs(upper - 1.0 / L - cdf)).max())


def histogram_edges(probs, n, bins, scale):
    """analytics.py:100-111: bin edges over x = 2^n p."""
    x = np.asarray(probs, dtype=np.float64).ravel() * 2.0 ** n
    top = float(x.max())
    if scale == "linear_Np":
        return np.linspace(0.0, top if top > 0 else 1.0, bins + 1)
    pos = x[x > 0]
    bottom = float(pos.min()) if pos.size else 1e-12
    top = top if top > bottom else bottom * 10
    return np.logspace(math.log10(bottom), math.log10(top), bins + 1)


def histogram(probs, n, bins=50, scale="linear_Np"):
    """analytics.py:90-121 -> (edges, density, pt_density)."""
    x = np.asarray(probs, dtype=np.float64).ravel() * 2.0 ** n
    edges = histogram_edges(probs, n, bins, scale)
    counts = np.histogram(x, bins=edges)[0]
    w = np.diff(edges)
    w = np.where(w > 0, w, 1.0)
    return edges, counts / (x.size * w), (np.exp(-edges[:-1]) - np.exp(-edges[1:])) / w


def postselect_curve(probs_desc, n, points=100):
    """analytics.py:124-143 -> [(fraction, xeb of the top k)]."""
    p = np.asarray(probs_desc, dtype=np.float64).ravel()
    L = p.size
    ks = sorted({1, L} | {max(1, math.ceil(L * i / points)) for i in range(1, points + 1)})
    c = np.cumsum(p)
    return [(k / L, (2.0 ** n / k) * float(c[k - 1]) - 1.0) for k in ks]


def mixed_xeb(known_probs, n, num_random):
    """analytics.py:146-156."""
    k = np.asarray(known_probs).size
    return 0.0 if k == 0 else k * xeb(known_probs, n)[1] / (k + num_random)


def marginal_and_conditional(probs, n2):
    """analytics.py:159-177 -> (marginal, conditional, xeb of the conditional)."""
    p = np.asarray(probs, dtype=np.float64).ravel()
    m = float(p.sum())
    cond = p / m
    return m, cond, xeb(cond, n2)[1]
