"""Device buffers (torch is used as the allocator only) + libtnb adds."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class DeviceAdder:
    """Upload host vectors and add them pairwise on the device through
    ``tnb_add_tree`` (same IEEE ops as numpy's elementwise ``a + b``)."""

    def __init__(self, dtype, elems: int, device: int):
        import torch

        self.torch = torch
        self.np_dtype = np.dtype(dtype)
        self.precision = _lib.TNB_SINGLE if self.np_dtype == np.complex64 else _lib.TNB_DOUBLE
        self.tdtype = torch.complex64 if self.precision == _lib.TNB_SINGLE else torch.complex128
        self.elems = int(elems)
        self.device = device
        self.dev = torch.device("cuda", device)

    def upload(self, host: np.ndarray):
        t = self.torch.from_numpy(np.ascontiguousarray(host, dtype=self.np_dtype))
        return t.to(self.dev)

    def add(self, a, b):
        out = self.torch.empty(self.elems, dtype=self.tdtype, device=self.dev)
        self.torch.cuda.synchronize(self.dev)
        ptrs = (C.c_void_p * 2)(a.data_ptr(), b.data_ptr())
        _lib.check(_lib.load().tnb_add_tree(self.device, self.precision, self.elems, 2, ptrs,
                                            C.c_void_p(out.data_ptr())))
        return out

    def download(self, t) -> np.ndarray:
        self.torch.cuda.synchronize(self.dev)
        return t.cpu().numpy()


def add_tree_device(tensors, out, device: int) -> None:
    """out = aligned binary-tree sum of equal-size torch CUDA tensors."""
    import torch

    precision = _lib.TNB_SINGLE if tensors[0].dtype == torch.complex64 else _lib.TNB_DOUBLE
    torch.cuda.synchronize(tensors[0].device)
    ptrs = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    _lib.check(_lib.load().tnb_add_tree(device, precision, tensors[0].numel(), len(tensors), ptrs,
                                        C.c_void_p(out.data_ptr())))
