"""Diagnostic: do kind::f16 UMMAs honour fp16 subnormal inputs?
A's row blocks are scaled by 2^-e; the fp16 scale comes from max|A| (block 0),
so the lo parts of the small blocks become subnormal.  With subnormals
honoured their relative error stays ~1e-6; flushed, it approaches 2^-11."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2103_03074_b200 import _lib
lib = _lib.load()
rng = np.random.default_rng(1)
M, N, K = 1024, 512, 1024
exps = [0, 4, 8, 12, 16, 20, 24]
blk = M // 8
A = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K)))
for i, e in enumerate(exps):
    A[i * blk:(i + 1) * blk] *= 2.0 ** -e
A = A.astype(np.complex64)
B = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
C = np.empty((M, N), np.complex64)
_lib.check(lib.tnb_cgemm(0, M, N, K, A.ctypes.data, B.ctypes.data, C.ctypes.data, 0, 1))
R = A.astype(np.complex128) @ B.astype(np.complex128)
for i, e in enumerate(exps):
    s = slice(i * blk, (i + 1) * blk)
    err = np.linalg.norm(C[s] - R[s]) / np.linalg.norm(R[s])
    print(f"row block scaled 2^-{e:2d}: rel err {err:.3e}")
