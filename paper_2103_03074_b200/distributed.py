"""Multi-GPU slice sharding (one process per GPU, torch.distributed/NCCL).

Slices are independent: rank r of N owns the
aligned contiguous slice range [a + r*w, a + (r+1)*w), w = (b-a)/N -- the
same layout as the reference's thread fan-out (cli.py:367-371).  Each rank
sums its range on its own device; the exchange is ONE collective:

* ``sharded_amplitudes`` -- every rank contracts the (linear) tail with its
  partial head vector and a single NCCL all-reduce(sum) combines the 2^n2
  amplitude partials (BASELINE north_star);
* ``sharded_head_vector(mode="fixed")`` -- all-gather of the partial head
  vectors, then the aligned binary-tree combine of ``reduce_partials``
  (engine.py:428-442) on the device: bit-identical to the single-GPU
  fixed-mode result.  ``mode="free"`` uses an all-reduce instead.

The partial computation and the add are injectable so the collective
choreography is testable with ``gloo`` on CPU (tests/test_distributed.py);
the defaults run libtnb on the rank's GPU.
"""

from __future__ import annotations

import dataclasses
import os

import numpy as np

from .errors import RangeOutOfBounds


def aligned_ranges(a: int, b: int, parts: int) -> list:
    """Split [a, b) into `parts` contiguous ranges; equal and aligned when
    parts is a power of two dividing b - a (required for bit-exact fixed mode)."""
    if parts <= 0:
        raise ValueError("parts must be positive")
    n = b - a
    if n < parts:
        raise RangeOutOfBounds(f"{n} slices cannot be split over {parts} ranks")
    base, extra = divmod(n, parts)
    out, lo = [], a
    for r in range(parts):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def tree_combine(items, add):
    """reduce_partials' aligned binary tree over equal-width ranges."""
    if len(items) == 1:
        return items[0]
    if len(items) & (len(items) - 1):
        acc = items[0]
        for x in items[1:]:
            acc = add(acc, x)
        return acc
    mid = len(items) // 2
    return add(tree_combine(items[:mid], add), tree_combine(items[mid:], add))


def _torch_add(x, y):
    return x + y


def _device_add(x, y):
    import torch

    from .device import add_tree_device

    if not x.is_cuda:
        return x + y
    out = torch.empty_like(x)
    add_tree_device([x, y], out, x.device.index)
    return out


def rank_device() -> int:
    """This rank's GPU: torch's current device, or LOCAL_RANK when the caller
    left the current device at 0 (torchrun starts every rank there); the
    choice is made current so torch, NCCL and libtnb all use it."""
    import torch

    cur = torch.cuda.current_device()
    lr = os.environ.get("LOCAL_RANK")
    if lr is not None and cur == 0 and 0 < int(lr) < torch.cuda.device_count():
        cur = int(lr)
        torch.cuda.set_device(cur)
    return cur


def _tdtype(precision):
    import torch

    return torch.complex64 if precision == "single" else torch.complex128


def _all_gather(flat, world, group):
    """all_gather of equal-size tensors.  NCCL gathers device buffers in
    place; gloo has no CUDA all_gather, so (gloo test runs only) the gather
    goes through host copies and the parts return to the device."""
    import torch
    import torch.distributed as dist

    if flat.is_cuda and dist.get_backend(group) == "gloo":
        host = flat.cpu()
        bufs = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(bufs, host, group=group)
        return [b.to(flat.device) for b in bufs]
    bufs = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(bufs, flat, group=group)
    return bufs


def _rank_world(group):
    import torch.distributed as dist

    return dist.get_rank(group), dist.get_world_size(group)


def sharded_head_vector(tn, tree, sliced_indices, s1, slice_range=None, precision="single",
                        mode="fixed", group=None, partial_fn=None, add=None):
    """Full head vector of [a, b) computed across the process group."""
    import torch
    import torch.distributed as dist

    from . import engine

    rank, world = _rank_world(group)
    n_e = len(sliced_indices)
    a, b = slice_range if slice_range is not None else (0, 1 << n_e)
    lo, hi = aligned_ranges(a, b, world)[rank]
    if partial_fn is None:
        # head partial stays on this rank's device (no host round trip)
        dev = rank_device()
        n_c = len(engine._split(tn, tree)[4])
        local = torch.empty(1 << n_c, dtype=_tdtype(precision), device=torch.device("cuda", dev))
        template = engine.head_vector_to_device(tn, tree, sliced_indices, s1, local,
                                                slice_range=(lo, hi), precision=precision,
                                                mode=mode, device=dev)
        add = add or _device_add
    else:
        local, template = partial_fn(lo, hi)
        add = add or _torch_add
    flat = torch.view_as_real(local).reshape(-1)
    if mode == "fixed":
        bufs = _all_gather(flat, world, group)
        parts = [torch.view_as_complex(x.reshape(-1, 2)) for x in bufs]
        total = tree_combine(parts, add)
    else:
        dist.all_reduce(flat, group=group)
        total = torch.view_as_complex(flat.reshape(-1, 2))
    data = total.cpu().numpy()
    return dataclasses.replace(template, data=data, slice_range=(a, b))


def sharded_amplitudes(tn, tree, sliced_indices, s1, slice_range=None, precision="single",
                       mode="fixed", group=None, partial_fn=None):
    """Amplitudes of the slice range with one all-reduce of the amplitude vector."""
    import torch
    import torch.distributed as dist

    from . import engine

    rank, world = _rank_world(group)
    n_e = len(sliced_indices)
    a, b = slice_range if slice_range is not None else (0, 1 << n_e)
    lo, hi = aligned_ranges(a, b, world)[rank]
    if partial_fn is None:
        # head -> tail -> all-reduce on the device; one D2H of the result
        dev = rank_device()
        cuda = torch.device("cuda", dev)
        n_c = len(engine._split(tn, tree)[4])
        n2 = len(tn.open_output_indices)
        head_dev = torch.empty(1 << n_c, dtype=_tdtype(precision), device=cuda)
        hv = engine.head_vector_to_device(tn, tree, sliced_indices, s1, head_dev,
                                          slice_range=(lo, hi), precision=precision,
                                          mode=mode, device=dev)
        local = torch.empty(1 << n2, dtype=_tdtype(precision), device=cuda)
        tab = engine.tail_amplitudes_to_device(tn, tree, hv, head_dev, local,
                                               precision=precision, device=dev)
    else:
        local, tab = partial_fn(lo, hi)
    flat = torch.view_as_real(local).reshape(-1)
    dist.all_reduce(flat, group=group)
    amps = torch.view_as_complex(flat.reshape(-1, 2)).cpu().numpy()
    want = np.complex64 if precision == "single" else np.complex128
    return dataclasses.replace(tab, amplitudes=amps.astype(want, copy=False))


def threaded_head_vector(tn, tree, sliced_indices, s1, slice_range=None, precision="single",
                         mode="fixed", devices=None):
    """Single-process multi-GPU ``compute_head_vector``: the aligned ranges
    of [a, b) (one per entry of ``devices``, default every visible GPU) run
    in one thread per device, and the partial head vectors are combined
    with ``reduce_partials``' aligned binary tree (engine.py:428-442) on the
    host -- in fixed mode bit-identical to one call over [a, b) when the
    device count is a power of two dividing b - a.  No torch.distributed
    needed (the reference's ``cli run --threads`` pattern, cli.py:367-380,
    without the file round trip)."""
    import concurrent.futures as cf

    from . import _lib, engine

    if devices is None:
        devices = list(range(max(1, _lib.device_count())))
    n_e = len(sliced_indices)
    a, b = slice_range if slice_range is not None else (0, 1 << n_e)
    spans = aligned_ranges(a, b, len(devices))

    def one(i):
        lo, hi = spans[i]
        return engine.compute_head_vector(tn, tree, sliced_indices, s1, slice_range=(lo, hi),
                                          precision=precision, mode=mode, device=devices[i])

    with cf.ThreadPoolExecutor(max_workers=len(devices)) as pool:
        parts = list(pool.map(one, range(len(devices))))
    if mode == "fixed":
        total = tree_combine([p.data for p in parts], lambda x, y: x + y)
    else:
        total = parts[0].data
        for p in parts[1:]:
            total = total + p.data
    return dataclasses.replace(parts[0], data=total, slice_range=(a, b))


class NcclComm:
    """The C-ABI collective (``tnb_allreduce_sum``, include/tnb.h) for callers
    that do not run torch.distributed: one communicator per process/device.
    The 128-byte NCCL id is created on rank 0 and shared by the caller
    (``unique_id()``; e.g. over any side channel or a gloo broadcast)."""

    def __init__(self, nranks: int, uid: bytes, rank: int, device: int = 0):
        import ctypes as C

        from . import _lib

        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self._lib = _lib
        buf = C.create_string_buffer(uid, 128)
        out = C.c_void_p()
        _lib.check(_lib.load().tnb_nccl_comm_create(nranks, C.addressof(buf), rank, device,
                                                    C.byref(out)))
        self.handle = out

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from . import _lib

        buf = C.create_string_buffer(128)
        _lib.check(_lib.load().tnb_nccl_unique_id(C.addressof(buf)))
        return buf.raw

    def allreduce_sum(self, tensor, stream=None) -> None:
        """In-place sum over ranks of a complex64/complex128 CUDA tensor."""
        import torch

        if not tensor.is_cuda or not tensor.is_contiguous():
            raise ValueError("allreduce_sum needs a contiguous CUDA tensor")
        prec = {torch.complex64: self._lib.TNB_SINGLE, torch.complex128: self._lib.TNB_DOUBLE}
        if tensor.dtype not in prec:
            raise ValueError("allreduce_sum takes complex64 or complex128")
        s = stream.cuda_stream if stream is not None else None
        self._lib.check(self._lib.load().tnb_allreduce_sum(self.handle, prec[tensor.dtype],
                                                           tensor.data_ptr(), tensor.numel(), s))

    def close(self) -> None:
        if self.handle:
            self._lib.check(self._lib.load().tnb_nccl_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
