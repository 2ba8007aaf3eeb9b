"""Bounded CPU timing of the reference head-slice contraction -- TEST/BENCH
INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and --impl reference arm).

A full C4 head slice takes ~214 s of numpy on 8 cores, too long
for a benchmark run.  This sampler times the reference's per-step operation
-- ``np.tensordot`` with the exact operand axis orders that
``_contract_steps`` (engine.py:117-144) produces for the slice -- on random
operands, step by step.  Steps whose full cost exceeds ``step_cap_s`` are
timed on 1/2^j of their shared-index range (j leading shared axes pinned)
and scaled by 2^j.  The estimate of one slice's time is the sum over all
steps.  Numbers are reported as a bounded sample, never as a full run.
"""

from __future__ import annotations

import os
import time

import numpy as np


def step_layouts(tn, leaves, steps, sliced):
    """Per step: (a_ids, b_ids, shared) exactly as engine.py:125-134 builds them."""
    ids = {}
    for nid in leaves:
        ids[nid] = [ix for ix in tn.nodes[nid].indices if ix not in sliced]
    out = []
    for s in steps:
        a, b = ids.pop(s.lhs), ids.pop(s.rhs)
        shared = [ix for ix in a if ix in b]
        out.append((a, b, shared))
        ids[s.out] = [ix for ix in a if ix not in b] + [ix for ix in b if ix not in a]
    return out


def _rand(shape, rng, dtype):
    n = int(np.prod(shape)) if shape else 1
    base = (rng.standard_normal(min(n, 1 << 16)) + 1j * rng.standard_normal(min(n, 1 << 16)))
    reps = -(-n // base.size)
    return np.tile(base.astype(dtype), reps)[:n].reshape(shape)


def _time_step(a_ids, b_ids, shared, pin_axes, j, rng, dtype):
    """Seconds of np.tensordot with the first j of ``pin_axes`` pinned."""
    pin = set(pin_axes[:j])
    a_axes = [ix for ix in a_ids if ix not in pin]
    b_axes = [ix for ix in b_ids if ix not in pin]
    sh = [ix for ix in shared if ix not in pin]
    A = _rand((2,) * len(a_axes), rng, dtype)
    B = _rand((2,) * len(b_axes), rng, dtype)
    t0 = time.perf_counter()
    if sh:
        np.tensordot(A, B, axes=([a_axes.index(x) for x in sh], [b_axes.index(x) for x in sh]))
    else:
        np.multiply.outer(A, B)
    return time.perf_counter() - t0


def time_head_slice(tn, tree, sliced, precision="single", rate_guess=5e11, step_cap_s=2.0,
                    seed=0, log=None):
    """Estimated seconds for one head slice + the sample description.

    Big steps are timed with j and j+1 leading free axes of their larger
    operand pinned; the per-call cost model t(j) = G / 2^j + F (G: work
    proportional to that range, F: fixed per-call cost such as transposing
    the other operand)
    gives the full-step estimate G + F from the two timings."""
    from .engine_np import split

    dtype = np.complex64 if precision == "single" else np.complex128
    rng = np.random.default_rng(seed)
    head_leaves, head_steps, _, _, _ = split(tn, tree)
    layouts = step_layouts(tn, head_leaves, head_steps, set(sliced))
    est = 0.0
    wall = 0.0
    scaled_steps = 0
    rate = rate_guess
    order = sorted(range(len(layouts)), key=lambda i: len(layouts[i][0]) + len(layouts[i][1]))
    for i in order:
        a_ids, b_ids, shared = layouts[i]
        mults = 2.0 ** (len(a_ids) + len(b_ids) - len(shared))
        # pin leading free axes of the larger operand: the GEMM work, that
        # operand's transposition and the result all scale with 1/2^j
        big, small = (a_ids, b_ids) if len(a_ids) >= len(b_ids) else (b_ids, a_ids)
        pin_axes = [ix for ix in big if ix not in small]
        j = 0
        while j + 1 < len(pin_axes) and 8 * mults / 2 ** j / rate > step_cap_s:
            j += 1
        t_j = _time_step(a_ids, b_ids, shared, pin_axes, j, rng, dtype)
        wall += t_j
        if j:
            t_j1 = _time_step(a_ids, b_ids, shared, pin_axes, j + 1, rng, dtype)
            wall += t_j1
            g = 2 ** (j + 1) * (t_j - t_j1)
            f = 2 * t_j1 - t_j
            step_est = min(max(g + max(f, 0.0), t_j), t_j * 2 ** j)
            scaled_steps += 1
        else:
            step_est = t_j
        est += step_est
        if 8 * mults / 2 ** j > 1e9 and t_j > 0:
            rate = 0.5 * rate + 0.5 * (8 * mults / 2 ** j / t_j)
        if log:
            log(f"step {i}: 2^{np.log2(mults):.1f} mults, pinned {j}: {t_j:.3f}s -> {step_est:.2f}s")
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or str(len(os.sched_getaffinity(0)))
    sample = (f"all {len(layouts)} head steps of one slice: np.tensordot (the reference op, "
              f"engine.py:129) on random operands with the slice's exact axis layouts; "
              f"{scaled_steps} large steps timed on 1/2^j and 1/2^(j+1) of their larger operand's free-index "
              f"range and extrapolated to the full range; {wall:.1f}s of CPU work sampled, "
              f"OpenBLAS threads={threads}")
    return est, wall, sample
