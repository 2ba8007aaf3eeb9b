"""On-device output-distribution analytics, drop-in for tncut analytics.py.

Same names, signatures, return types and exceptions as the reference
(analytics.py:26-177); the reductions run in libtnb.so on the device
(``tnb_prob_*``, include/tnb.h).  Inputs are either plain probability arrays
(the reference's calling convention; uploaded once) or device-resident
torch tensors -- probabilities (float64) or amplitudes (complex64/128, turned
into |a|^2 on the device) -- so a tail result never has to leave HBM.

Numerics: sums are fp64 with a fixed reduction tree (deterministic, within
~1e-15 relative of numpy's pairwise sum); min/max, histogram counts and the
post-selection order are exact.  Probabilities derived on the device from
complex64 amplitudes are computed in fp64 (the reference's
``np.abs(c64)**2`` rounds to fp32 first; the difference is <= 2^-23
relative per element).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

try:  # the reference's own report/row types and exceptions when importable
    from tncut.analytics import HistogramRow, XebReport  # type: ignore
    from tncut.errors import EmptyInput, IncompleteEnumeration, NotSorted, ZeroMarginal  # type: ignore
except Exception:  # pragma: no cover - tncut absent (e.g. the GPU box)
    from .errors import TncutError

    class EmptyInput(TncutError):
        pass

    class NotSorted(TncutError):
        pass

    class IncompleteEnumeration(TncutError):
        pass

    class ZeroMarginal(TncutError):
        pass

    @dataclass
    class XebReport:  # analytics.py:26-43
        L: int
        n: int
        f_xeb: float
        p_min: float
        p_max: float
        notes: str = ""

        def doc(self) -> dict:
            return {"L": self.L, "n": self.n, "f_xeb": self.f_xeb, "p_min": self.p_min,
                    "p_max": self.p_max, "notes": self.notes}

    @dataclass
    class HistogramRow:  # analytics.py:82-87
        bin_lo: float
        bin_hi: float
        density: float
        pt_density: float


_device = None  # None: torch's current device (the rank's GPU under torchrun)


def set_device(device) -> None:
    """Device for host (numpy) inputs; None = torch's current device."""
    global _device
    _device = None if device is None else int(device)


class _DevProbs:
    """A float64 probability vector in device memory (owned torch tensor)."""

    def __init__(self, probs, copy: bool = False):
        import torch

        _lib.require_device()
        self.lib = _lib.load()
        if isinstance(probs, torch.Tensor) and probs.is_cuda:
            self.device = probs.device.index
            if probs.is_complex():
                amps = probs.contiguous()
                prec = _lib.TNB_SINGLE if amps.dtype == torch.complex64 else _lib.TNB_DOUBLE
                self.t = torch.empty(amps.numel(), dtype=torch.float64, device=amps.device)
                torch.cuda.synchronize(amps.device)
                if amps.numel():
                    _lib.check(self.lib.tnb_probabilities(self.device, prec, C.c_void_p(amps.data_ptr()),
                                                          amps.numel(), C.c_void_p(self.t.data_ptr())))
            else:
                t = probs.reshape(-1).to(torch.float64)
                self.t = t.clone() if (copy and t.data_ptr() == probs.data_ptr()) else t.contiguous()
        else:
            host = np.ascontiguousarray(np.asarray(probs, dtype=float).reshape(-1))
            self.device = _device if _device is not None else torch.cuda.current_device()
            self.t = torch.from_numpy(host).to(torch.device("cuda", self.device))
        torch.cuda.synchronize(self.t.device)
        self.n = int(self.t.numel())

    @property
    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def reduce(self):
        """(sum, min, max, min over p > 0 -- inf when none)."""
        out = (C.c_double * 4)()
        _lib.check(self.lib.tnb_prob_reduce(self.device, self.ptr, self.n, out))
        return float(out[0]), float(out[1]), float(out[2]), float(out[3])

    def sort(self, descending: bool) -> None:
        _lib.check(self.lib.tnb_prob_sort(self.device, self.ptr, self.n, 1 if descending else 0))

    def is_sorted_desc(self) -> bool:
        ok = C.c_int32(0)
        _lib.check(self.lib.tnb_prob_is_sorted_desc(self.device, self.ptr, self.n, C.byref(ok)))
        return bool(ok.value)

    def prefix_sums(self, ks) -> np.ndarray:
        ks = np.ascontiguousarray(ks, dtype=np.int64)
        out = np.empty(ks.size, dtype=np.float64)
        _lib.check(self.lib.tnb_prob_prefix_sums(
            self.device, self.ptr, self.n, ks.ctypes.data_as(C.POINTER(C.c_int64)), ks.size,
            out.ctypes.data_as(C.POINTER(C.c_double))))
        return out


def xeb(probs, n: int, notes: str = "") -> XebReport:
    """Linear XEB (2^n / L) * sum(p) - 1 (analytics.py:46-58)."""
    d = _DevProbs(probs)
    if d.n == 0:
        raise EmptyInput("xeb needs at least one probability")
    s, lo, hi, _ = d.reduce()
    return XebReport(L=d.n, n=n, f_xeb=(2.0 ** n / d.n) * s - 1.0, p_min=lo, p_max=hi, notes=notes)


def porter_thomas_density(p: float, n: int) -> float:  # analytics.py:61-62
    return 2.0 ** n * math.exp(-p * 2.0 ** n)


def porter_thomas_sample(n: int, size: int, rng) -> np.ndarray:  # analytics.py:65-67
    return rng.exponential(scale=2.0 ** -n, size=size)


def ks_to_porter_thomas(probs, n: int) -> float:
    """KS distance of 2^n p against Exp(1) (analytics.py:70-79): device sort
    + one max reduction."""
    d = _DevProbs(probs, copy=True)
    if d.n == 0:
        raise EmptyInput("no probabilities")
    d.sort(descending=False)
    out = C.c_double(0.0)
    _lib.check(d.lib.tnb_prob_ks(d.device, d.ptr, d.n, 2.0 ** n, C.byref(out)))
    return float(out.value)


def histogram(probs, n: int, bins: int = 50, scale: str = "linear_Np"):
    """Density of x = 2^n p with the Porter-Thomas overlay (analytics.py:90-121);
    the edges follow the reference exactly, the binning runs on the device."""
    d = _DevProbs(probs)
    if d.n == 0:
        raise EmptyInput("no probabilities")
    if bins < 1:
        raise ValueError("bins must be >= 1")
    _, _, hi_p, lo_pos = d.reduce()
    hi = float(hi_p * 2.0 ** n)
    if scale == "linear_Np":
        edges = np.linspace(0.0, hi if hi > 0 else 1.0, bins + 1)
    elif scale == "log":
        lo = float(lo_pos * 2.0 ** n) if math.isfinite(lo_pos) else 1e-12
        hi = hi if hi > lo else lo * 10
        edges = np.logspace(math.log10(lo), math.log10(hi), bins + 1)
    else:
        raise ValueError(f"unknown scale {scale!r}")
    edges = np.ascontiguousarray(edges, dtype=np.float64)
    counts = np.zeros(bins, dtype=np.int64)
    _lib.check(d.lib.tnb_prob_histogram(d.device, d.ptr, d.n, 2.0 ** n,
                                        edges.ctypes.data_as(C.POINTER(C.c_double)), bins,
                                        counts.ctypes.data_as(C.POINTER(C.c_int64))))
    widths = np.diff(edges)
    density = counts / (d.n * np.where(widths > 0, widths, 1.0))
    pt_mass = np.exp(-edges[:-1]) - np.exp(-edges[1:])
    pt_density = pt_mass / np.where(widths > 0, widths, 1.0)
    return [HistogramRow(float(edges[i]), float(edges[i + 1]), float(density[i]), float(pt_density[i]))
            for i in range(bins)]


def postselect_curve(probs_desc, n: int, points: int = 100):
    """XEB of the top fraction of bitstrings (analytics.py:124-143); the input
    must be sorted descending (``sort_desc`` sorts on the device)."""
    d = _DevProbs(probs_desc)
    if d.n == 0:
        raise EmptyInput("no probabilities")
    if not d.is_sorted_desc():
        raise NotSorted("probabilities must be sorted descending")
    L = d.n
    ks = sorted({1, L} | {max(1, math.ceil(L * i / points)) for i in range(1, points + 1)})
    sums = d.prefix_sums(ks)
    return [(k / L, (2.0 ** n / k) * float(c) - 1.0) for k, c in zip(ks, sums)]


def sort_desc(probs):
    """Device-resident probabilities sorted descending (torch float64 tensor),
    the caller-side sort postselect_curve expects."""
    d = _DevProbs(probs, copy=True)
    d.sort(descending=True)
    return d.t


def mixed_xeb(known_probs, n: int, num_random: int) -> float:
    """Expected XEB after mixing with uniform-random bitstrings (analytics.py:146-156)."""
    import torch

    k = int(known_probs.numel()) if isinstance(known_probs, torch.Tensor) else int(np.asarray(known_probs).size)
    if k == 0 and num_random == 0:
        raise EmptyInput("nothing to mix")
    if k == 0:
        return 0.0
    f_known = xeb(known_probs, n).f_xeb
    return k * f_known / (k + num_random)


def marginal_and_conditional(table):
    """P(s1), the conditional distribution over s2 and its XEB
    (analytics.py:159-177).  ``table.amplitudes`` may be a host array or a
    device tensor; the conditional vector is returned on the same side."""
    import torch

    amps = table.amplitudes
    on_dev = isinstance(amps, torch.Tensor) and amps.is_cuda
    d = _DevProbs(amps if on_dev else np.asarray(table.probabilities, dtype=float))
    n2 = len(table.open_qubits)
    if d.n != 1 << n2:
        raise IncompleteEnumeration(f"{d.n} rows but 2^{n2} assignments expected")
    marginal = d.reduce()[0]
    if marginal == 0.0:
        raise ZeroMarginal("P(s1) = 0; conditional undefined")
    cond = d.t / marginal
    f = xeb(cond, n2).f_xeb
    return marginal, (cond if on_dev else cond.cpu().numpy()), f
