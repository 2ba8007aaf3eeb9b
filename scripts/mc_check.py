"""Correctness of the A-multicast GEMM variant (TNB_GEMM_MC=1) vs fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2103_03074_b200 import _lib
lib = _lib.load()
rng = np.random.default_rng(0)
for (M, N, K) in [(1 << 12, 1 << 11, 1 << 10), (1 << 13, 1 << 9, 1 << 8), (1 << 12, 1 << 7, 1 << 11), (1 << 14, 1 << 12, 1 << 12)]:
    A = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))).astype(np.complex64)
    B = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    C = np.empty((M, N), np.complex64)
    _lib.check(lib.tnb_cgemm(0, M, N, K, A.ctypes.data, B.ctypes.data, C.ctypes.data, 0, 1))
    R = A[:512].astype(np.complex128) @ B.astype(np.complex128)
    e = np.linalg.norm(C[:512] - R) / np.linalg.norm(R)
    R2 = A[-512:].astype(np.complex128) @ B.astype(np.complex128)
    e2 = np.linalg.norm(C[-512:] - R2) / np.linalg.norm(R2)
    print(f"M={M} N={N} K={K}: rel err head {e:.2e} tail {e2:.2e}", flush=True)
