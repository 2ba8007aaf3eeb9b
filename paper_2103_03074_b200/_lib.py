"""ctypes binding of libtnb.so (include/tnb.h).

There is no CPU fallback: importing the engine on a machine where the
library is missing raises, and every compute entry point raises when no
sm_100 device is present.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtnb.so")

TNB_OK, TNB_ERR_ARG, TNB_ERR_SHAPE, TNB_ERR_RANGE, TNB_ERR_CUDA, TNB_ERR_NOMEM, TNB_ERR_NODEV = range(7)
TNB_DOUBLE, TNB_SINGLE = 0, 1
TNB_FIXED, TNB_FREE = 0, 1
TNB_FLAG_NO_TENSOR_CORES = 0x1
TNB_FLAG_NO_HOIST = 0x2
TNB_FLAG_REUSE_SLICES = 0x4
TNB_FLAG_NO_FUSE = 0x8

i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
P = C.c_void_p


class ProgramDesc(C.Structure):
    _fields_ = [
        ("n_leaves", i32), ("leaf_ids", C.POINTER(i64)), ("leaf_ranks", C.POINTER(i32)),
        ("leaf_indices", C.POINTER(i64)), ("leaf_data", C.POINTER(f64)),
        ("n_steps", i32), ("steps", C.POINTER(i64)),
        ("n_sliced", i32), ("sliced", C.POINTER(i64)),
        ("n_out", i32), ("out_order", C.POINTER(i64)),
        ("precision", i32), ("device", i32), ("flags", u32),
    ]


class ProgramInfo(C.Structure):
    _fields_ = [
        ("out_elems", i64), ("flops_per_slice", f64), ("tc_flops_per_slice", f64),
        ("arena_bytes", i64), ("persistent_bytes", i64), ("scratch_bytes", i64),
        ("n_steps_tc", i32), ("n_steps_simt", i32), ("n_steps_hoisted", i32),
        ("kernels_per_slice", i32), ("reuse_bytes", i64),
        ("n_steps_fused", i32), ("n_steps_fused_fast", i32),
    ]


class Timing(C.Structure):
    _fields_ = [
        ("total_ms", f64), ("gemm_ms", f64), ("convert_ms", f64), ("simt_ms", f64),
        ("other_ms", f64), ("launches", i64), ("gemm_launches", i64), ("gemm_flops", f64),
        ("steps_reused", i64), ("scale_redos", i64),
    ]


EXPORTS = {
    "tnb_abi_version": (i32, []),
    "tnb_last_error": (C.c_char_p, []),
    "tnb_device_count": (i32, [C.POINTER(i32)]),
    "tnb_program_create": (i32, [C.POINTER(ProgramDesc), C.POINTER(P)]),
    "tnb_program_destroy": (i32, [P]),
    "tnb_program_get_info": (i32, [P, C.POINTER(ProgramInfo)]),
    "tnb_program_set_leaf": (i32, [P, i32, C.POINTER(f64)]),
    "tnb_program_set_leaf_device": (i32, [P, i32, P]),
    "tnb_program_set_leaves": (i32, [P, i32, C.POINTER(i32), C.POINTER(f64)]),
    "tnb_program_set_leaf_c64": (i32, [P, i32, C.POINTER(C.c_float)]),
    "tnb_program_run_range": (i32, [P, u64, u64, i32, P, i32]),
    "tnb_program_set_timing": (i32, [P, i32]),
    "tnb_program_get_timing": (i32, [P, C.POINTER(Timing)]),
    "tnb_cgemm": (i32, [i32, i64, i64, i64, P, P, P, i32, i32]),
    "tnb_add_tree": (i32, [i32, i32, i64, i32, C.POINTER(P), P]),
    "tnb_probabilities": (i32, [i32, i32, P, i64, P]),
    "tnb_prob_reduce": (i32, [i32, P, i64, C.POINTER(f64)]),
    "tnb_prob_histogram": (i32, [i32, P, i64, f64, C.POINTER(f64), i32, C.POINTER(i64)]),
    "tnb_prob_sort": (i32, [i32, P, i64, i32]),
    "tnb_prob_is_sorted_desc": (i32, [i32, P, i64, C.POINTER(i32)]),
    "tnb_prob_prefix_sums": (i32, [i32, P, i64, C.POINTER(i64), i32, C.POINTER(f64)]),
    "tnb_prob_ks": (i32, [i32, P, i64, f64, C.POINTER(f64)]),
    "tnb_nccl_unique_id": (i32, [P]),
    "tnb_nccl_comm_create": (i32, [i32, P, i32, i32, C.POINTER(C.c_void_p)]),
    "tnb_nccl_comm_destroy": (i32, [C.c_void_p]),
    "tnb_allreduce_sum": (i32, [C.c_void_p, i32, C.c_void_p, i64, C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load libtnb.so once; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2103_03074_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tnb_abi_version() != 2:
            raise ImportError("libtnb.so ABI version mismatch")
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status == TNB_OK:
        return
    msg = load().tnb_last_error().decode(errors="replace")
    if status == TNB_ERR_SHAPE:
        raise errors.ShapeMismatch(msg)
    if status == TNB_ERR_RANGE:
        raise errors.RangeOutOfBounds(msg)
    if status == TNB_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"libtnb: {msg} (status {status})")


def device_count() -> int:
    n = i32(0)
    check(load().tnb_device_count(C.byref(n)))
    return n.value


def require_device() -> None:
    if device_count() == 0:
        raise RuntimeError("no CUDA device: the B200 executor has no CPU fallback")
