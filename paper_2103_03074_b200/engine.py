"""Drop-in replacement of the reference execution engine (tncut engine.py).

Same names, signatures, argument meaning, return types and exceptions as
``tncut.engine`` (engine.py:147-165, 242-378, 398-458); the arithmetic runs
in libtnb.so on an sm_100 device:

* ``compute_head_vector`` -> one compiled *program* per (head topology,
  slicing, precision, device), executed over the slice range in C++/CUDA
  (sliced-leaf gather, per-step tcgen05 or SIMT contraction, on-device
  fixed/free slice sum, root permuted to ascending cut ids);
* ``compute_tail_amplitudes`` -> the head vector is absorbed into the tail
  network as one extra leaf and the result contracted on the device with
  the open indices kept (mathematically the reference's per-block
  ``T @ v_head``, engine.py:358-377, at 10^3-10^4x fewer multiplications);
  the amplitude rows keep the reference's s2 order (MSB = lowest open qubit);
* ``contract_tree`` -> the same program path with every index pinned;
* ``reduce_partials`` -> the reference's validation and aligned binary
  combine (engine.py:398-452), adds executed on the device.

``EngineStats`` is filled with the reference's exact counters, computed
analytically from the index sets (they depend only on the schedule).
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import hashlib
import os
import threading

import numpy as np

from . import _lib
from .errors import (BlockTooWide, ProvenanceMismatch, RangeGap, RangeOutOfBounds, RangeOverlap,
                     ShapeMismatch)
from .planner import cluster_small_steps, split, step_mults
from .provenance import circuit_sha, normalize_s1, order_sha256, provenance_hash
from .types import AmplitudeTable, EngineStats, HeadVector

DTYPES = {"double": np.complex128, "single": np.complex64}
_PREC = {"double": _lib.TNB_DOUBLE, "single": _lib.TNB_SINGLE}
_MODES = {"fixed": _lib.TNB_FIXED, "free": _lib.TNB_FREE}

# default device for the calling process (one process per GPU)
_default_device = 0
_flags = 0


def set_device(device: int) -> None:
    global _default_device
    _default_device = int(device)


_thread_devices = False
_thread_local = threading.local()
_thread_counter = [0]
_thread_lock = threading.Lock()


def set_thread_devices(on: bool) -> None:
    """Bind each calling thread to its own device, round-robin over the
    visible GPUs (first call of a thread picks the next one).  The
    reference's ``cli run --threads T`` fans ranges out over T threads
    (cli.py:367-380); with this on, those threads spread over the box's
    GPUs instead of queueing on device 0.  Off: every call uses
    ``set_device``'s device."""
    global _thread_devices
    _thread_devices = bool(on)


def _resolve_device(device):
    if device is not None:
        return int(device)
    if not _thread_devices:
        return _default_device
    dev = getattr(_thread_local, "device", None)
    if dev is None:
        n = max(1, _lib.device_count())
        with _thread_lock:
            dev = (_default_device + _thread_counter[0]) % n
            _thread_counter[0] += 1
        _thread_local.device = dev
    return dev


_reorder = os.environ.get("TNB_REORDER", "0") not in ("", "0")
_reorder_cache: dict = {}


def set_reorder(on: bool) -> None:
    """Opt-in: execute every head slice with a re-ordered head tree for the
    SAME sliced set (``treeopt.select_slices_b200(keep_slices=True,
    objective="b200")``, cached per plan).  The partial head vectors are the
    same (same masks; fp32 rounding differs like any other order), so is
    the API: ``HeadVector``, provenance and the ``EngineStats`` counters
    still describe the caller's tree (engine.py:138-140).  C4: 29.8x the
    slices/s of the reference tree (bench ``reordered_same_slices``)."""
    global _reorder
    _reorder = bool(on)


_slice_batch = int(os.environ.get("TNB_SLICE_BATCH", "0") or 0)


def set_slice_batch(k: int) -> None:
    """Opt-in: ``compute_head_vector`` contracts 2^k aligned slices per pass
    (``slice_batch.py``: the k lowest-mask-bit sliced indices un-sliced, tree
    re-ordered) whenever ``slice_range`` is 2^k-aligned; other ranges take
    the per-slice path.  Same HeadVector / provenance / counters; the sum
    inside a block is the contraction's, so results equal the per-slice
    path within fp32 rounding.  C4, k = 4: 1140 slices/s (bench
    ``batched_slices``)."""
    global _slice_batch
    _slice_batch = max(0, int(k))


_cluster_all = os.environ.get("TNB_CLUSTER_ALL", "0") == "1"


def _exec_head_steps(tn, tree, head_leaves, head_steps, sliced):
    """The head steps the program runs: the caller's (optionally with their
    tiny steps clustered into waves, TNB_CLUSTER_ALL=1), or (set_reorder) the
    re-ordered ones, never above the caller's largest intermediate."""
    if not _reorder or not head_steps or tree.first_cut is None:
        if _cluster_all and head_steps:
            sets = {n: tn.nodes[n].indices for n in head_leaves}
            return cluster_small_steps(sets, head_steps, frozenset(sliced))
        return head_steps
    key = hashlib.sha256(repr((tuple((n, tuple(tn.nodes[n].indices)) for n in head_leaves),
                               tuple(_steps_tuples(head_steps)), tuple(sliced))).encode()).hexdigest()
    hit = _reorder_cache.get(key)
    if hit is None:
        from . import treeopt

        sets = {n: tn.nodes[n].indices for n in head_leaves}
        _, sc = step_mults(sets, head_steps, frozenset(sliced))
        sc = max([sc] + [len(set(tn.nodes[n].indices) - set(sliced)) for n in head_leaves])
        plan, new_tree = treeopt.select_slices_b200(tn, tree, sc, objective="b200",
                                                    keep_slices=True, initial_slices=list(sliced))
        if list(plan.sliced_indices) != list(sliced):
            raise ShapeMismatch("re-ordering changed the sliced set")
        hit = new_tree.head_steps()
        if os.environ.get("TNB_CLUSTER", "1") != "0":
            hit = cluster_small_steps(sets, hit, frozenset(sliced))
        _reorder_cache[key] = hit
    return hit


def set_flags(flags: int) -> None:
    """Executor flags (``_lib.TNB_FLAG_*``) for programs compiled afterwards."""
    global _flags
    _flags = int(flags)


# ---------------------------------------------------------------------------
# Program wrapper

class Program:
    """A compiled contraction schedule living on one device (libtnb program)."""

    def __init__(self, leaves, steps, sliced, out_order, precision: str, device: int,
                 flags: int = 0):
        lib = _lib.load()
        _lib.require_device()
        self.lib = lib
        self.precision = precision
        self.device = device
        self.dtype = DTYPES[precision]
        self.n_leaves = len(leaves)
        self.leaf_pos = {nid: i for i, (nid, _, _) in enumerate(leaves)}
        self._leaf_data = [np.ascontiguousarray(d, dtype=np.complex128).reshape(-1)
                           for (_, _, d) in leaves]
        ids = np.array([nid for (nid, _, _) in leaves], dtype=np.int64)
        ranks = np.array([len(ix) for (_, ix, _) in leaves], dtype=np.int32)
        idx = np.array([i for (_, ix, _) in leaves for i in ix] or [0], dtype=np.int64)
        data = np.concatenate(self._leaf_data) if leaves else np.zeros(1, np.complex128)
        data = np.ascontiguousarray(data).view(np.float64)
        st = np.array([v for s in steps for v in s] or [0], dtype=np.int64)
        sl = np.array(list(sliced) or [0], dtype=np.int64)
        oo = np.array(list(out_order) or [0], dtype=np.int64)
        self._keep = (ids, ranks, idx, data, st, sl, oo)
        d = _lib.ProgramDesc(
            n_leaves=len(leaves),
            leaf_ids=ids.ctypes.data_as(C.POINTER(C.c_int64)),
            leaf_ranks=ranks.ctypes.data_as(C.POINTER(C.c_int32)),
            leaf_indices=idx.ctypes.data_as(C.POINTER(C.c_int64)),
            leaf_data=data.ctypes.data_as(C.POINTER(C.c_double)),
            n_steps=len(steps), steps=st.ctypes.data_as(C.POINTER(C.c_int64)),
            n_sliced=len(sliced), sliced=sl.ctypes.data_as(C.POINTER(C.c_int64)),
            n_out=len(out_order), out_order=oo.ctypes.data_as(C.POINTER(C.c_int64)),
            precision=_PREC[precision], device=device, flags=flags,
        )
        h = C.c_void_p()
        _lib.check(lib.tnb_program_create(C.byref(d), C.byref(h)))
        self.handle = h
        self.lock = threading.Lock()
        info = _lib.ProgramInfo()
        _lib.check(lib.tnb_program_get_info(self.handle, C.byref(info)))
        self.info = info
        _warm_pinned(info.out_elems, self.dtype)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.tnb_program_destroy(h)
            except Exception:
                pass

    def update_leaves(self, leaves) -> None:
        """Upload leaves whose values changed (repin), topology unchanged --
        one batched, staged upload through tnb_program_set_leaves."""
        with self.lock:
            self._update_leaves(leaves)

    def run(self, leaves, a: int, b: int, mode: str = "fixed", out=None, device_leaves=None):
        """Upload ``leaves`` (and bind ``device_leaves`` {pos: device ptr}) and
        run [a, b) as ONE critical section: programs are cached per topology
        and shared between threads (the reference's ``cli run --threads``
        fans compute_head_vector out over disjoint ranges, cli.py:367-380),
        so two callers with different s1 must not interleave their uploads
        with each other's runs."""
        with self.lock:
            self._update_leaves(leaves)
            for pos, ptr in (device_leaves or {}).items():
                _lib.check(self.lib.tnb_program_set_leaf_device(self.handle, pos, C.c_void_p(ptr)))
                self._leaf_data[pos] = None
            return self._run_range(a, b, mode, out)

    def _update_leaves(self, leaves) -> None:
        pos_list, datas = [], []
        for nid, _, d in leaves:
            pos = self.leaf_pos[nid]
            d = np.asarray(d)
            if d.size >= (1 << 16):
                # big leaves (the tail's head vector): upload unconditionally,
                # straight from complex64 when the program is single precision
                if self.precision == "single" and d.dtype == np.complex64:
                    buf = np.ascontiguousarray(d).reshape(-1).view(np.float32)
                    _lib.check(self.lib.tnb_program_set_leaf_c64(
                        self.handle, pos, buf.ctypes.data_as(C.POINTER(C.c_float))))
                    self._leaf_data[pos] = None
                    continue
            else:
                old = self._leaf_data[pos]
                if old is not None and d.size == old.size and np.array_equal(d.reshape(-1), old):
                    continue
            new = np.ascontiguousarray(d, dtype=np.complex128).reshape(-1)
            pos_list.append(pos)
            datas.append(new)
            self._leaf_data[pos] = new
        if not pos_list:
            return
        posv = np.asarray(pos_list, dtype=np.int32)
        flat = np.concatenate(datas).view(np.float64)
        _lib.check(self.lib.tnb_program_set_leaves(
            self.handle, len(pos_list), posv.ctypes.data_as(C.POINTER(C.c_int32)),
            flat.ctypes.data_as(C.POINTER(C.c_double))))

    def set_leaf_device(self, pos: int, dev_ptr: int) -> None:
        with self.lock:
            _lib.check(self.lib.tnb_program_set_leaf_device(self.handle, pos, C.c_void_p(dev_ptr)))
            self._leaf_data[pos] = None  # unknown host copy: force upload next time

    def run_range(self, a: int, b: int, mode: str = "fixed", out=None) -> np.ndarray:
        """Host result (numpy) unless ``out`` is a device pointer (int)."""
        with self.lock:
            return self._run_range(a, b, mode, out)

    def _run_range(self, a, b, mode, out):
        """run_range without the lock (callers hold it)."""
        if out is None:
            res = _host_array(self.info.out_elems, self.dtype)
            _lib.check(self.lib.tnb_program_run_range(
                self.handle, a, b, _MODES[mode], res.ctypes.data_as(C.c_void_p), 0))
            return res
        _lib.check(self.lib.tnb_program_run_range(
            self.handle, a, b, _MODES[mode], C.c_void_p(out), 1))
        return None

    def set_timing(self, on) -> None:
        """False/0 off, True/1 every kernel class, 2 GEMM launches + total only."""
        mode = (1 if on else 0) if isinstance(on, bool) else int(on)
        _lib.check(self.lib.tnb_program_set_timing(self.handle, mode))

    def timing(self) -> dict:
        t = _lib.Timing()
        _lib.check(self.lib.tnb_program_get_timing(self.handle, C.byref(t)))
        return {f: getattr(t, f) for f, _ in _lib.Timing._fields_}


_PIN_MIN_BYTES = 1 << 20


def _host_array(n: int, dtype) -> np.ndarray:
    """Result buffer for a device->host copy: page-locked (pinned) host memory
    for large results -- the copy then runs at full PCIe/C2C speed instead of
    through the driver's pageable staging -- exposed as a plain numpy array
    (the torch tensor owning the pinned block is kept alive as its base)."""
    nbytes = int(n) * np.dtype(dtype).itemsize
    if nbytes >= _PIN_MIN_BYTES:
        try:
            import torch

            tdt = torch.complex64 if np.dtype(dtype) == np.complex64 else torch.complex128
            return torch.empty(int(n), dtype=tdt, pin_memory=True).numpy()
        except Exception:  # pinning is an optimisation only
            pass
    return np.empty(int(n), dtype=dtype)


def _warm_pinned(n: int, dtype, blocks: int = 3) -> None:
    """Page-lock a few result-sized blocks once (program creation) and hand
    them to torch's pinned-memory cache, so the per-call result buffers of
    ``_host_array`` are cache hits instead of ~10 ms cudaHostAlloc calls (a
    new result is requested while the caller still holds the previous one)."""
    if int(n) * np.dtype(dtype).itemsize < _PIN_MIN_BYTES:
        return
    held = [_host_array(n, dtype) for _ in range(blocks)]
    del held


_cache: dict = {}
_cache_lock = threading.Lock()
_CACHE_MAX = 8


def _signature(leaves, steps, sliced, out_order, precision, device, flags) -> str:
    h = hashlib.sha256()
    for nid, ix, _ in leaves:
        h.update(repr((nid, tuple(ix))).encode())
    h.update(repr(tuple(tuple(s) for s in steps)).encode())
    h.update(repr((tuple(sliced), tuple(out_order), precision, device, flags)).encode())
    return h.hexdigest()


def get_program(leaves, steps, sliced, out_order, precision, device=None, flags=None,
                upload: bool = True) -> Program:
    """The cached program for this topology; ``upload`` puts ``leaves``' values
    on it (single-threaded callers).  Engine calls pass upload=False and run
    through ``Program.run`` so upload and run are one critical section."""
    device = _resolve_device(device)
    flags = _flags if flags is None else flags
    key = _signature(leaves, steps, sliced, out_order, precision, device, flags)
    with _cache_lock:
        prog = _cache.get(key)
        if prog is None:
            if len(_cache) >= _CACHE_MAX:
                _cache.pop(next(iter(_cache)))
            try:
                prog = Program(leaves, steps, sliced, out_order, precision, device, flags)
            except RuntimeError as exc:
                if "out of memory" not in str(exc) or not _cache:
                    raise
                # cached programs hold their arenas (tens of GB at 2^30 plans):
                # evict them and retry once
                _cache.clear()
                import gc

                gc.collect()
                prog = Program(leaves, steps, sliced, out_order, precision, device, flags)
            _cache[key] = prog
        else:
            _cache[key] = _cache.pop(key)  # LRU touch
    if upload:
        prog.update_leaves(leaves)
    return prog


def clear_cache() -> None:
    with _cache_lock:
        _cache.clear()


_split_cache: dict = {}


def _topology_key(tn, tree) -> tuple:
    """What ``split`` and the tail order depend on: the tree's steps and every
    node's index list -- not leaf values, so every ``repin`` of a network
    (one per s1) shares one entry."""
    return (tuple((s.lhs, s.rhs, s.out) for s in tree.steps), tree.first_cut,
            tuple((nid, tuple(tn.nodes[nid].indices)) for nid in sorted(tn.nodes)))


def _split(tn, tree):
    """planner.split memoised per topology (``_topology_key``): repeated calls
    (slice ranges, tail after head, an s1 sweep) reuse one split."""
    key = _topology_key(tn, tree)
    hit = _split_cache.get(key)
    if hit is not None:
        return hit
    res = split(tn, tree)
    with _cache_lock:
        if len(_split_cache) >= 16:
            _split_cache.pop(next(iter(_split_cache)))
        _split_cache[key] = res
    return res


def _steps_tuples(steps):
    return [(s.lhs, s.rhs, s.out) for s in steps]


def _leaf_entries(tn, leaf_ids):
    return [(nid, list(tn.nodes[nid].indices), tn.nodes[nid].data) for nid in leaf_ids]


# ---------------------------------------------------------------------------
# Reference-shaped API

def head_program(tn, tree, sliced_indices, precision="single", device=None, flags=None):
    """The compiled head program (for benchmarks / timing introspection)."""
    head_leaves, head_steps, _, _, cut = _split(tn, tree)
    run_steps = _exec_head_steps(tn, tree, head_leaves, head_steps, list(sliced_indices))
    return get_program(_leaf_entries(tn, head_leaves), _steps_tuples(run_steps),
                       list(sliced_indices), sorted(cut), precision, device, flags)


def compute_head_vector(tn, tree, sliced_indices, s1, slice_range=None, precision="double",
                        mode="fixed", stats=None, device=None) -> HeadVector:
    """Sum of head contractions over a slice range (engine.py:242-310)."""
    return _head(tn, tree, sliced_indices, s1, slice_range, precision, mode, stats, device, None)


def head_vector_to_device(tn, tree, sliced_indices, s1, out, slice_range=None,
                          precision="single", mode="fixed", stats=None, device=None) -> HeadVector:
    """``compute_head_vector`` whose 2^n_c result stays in device memory: it is
    written to ``out`` (a caller-owned contiguous torch CUDA tensor of the
    precision's complex dtype on ``device``; the call returns after the device
    finished).  The returned HeadVector carries the metadata with
    ``data=None``.  Used by the sharded (multi-GPU) path so head -> tail ->
    all-reduce never round-trips through the host."""
    _check_out(out, precision)
    return _head(tn, tree, sliced_indices, s1, slice_range, precision, mode, stats, device,
                 out, batch_ok=False)


def _check_out(t, precision):
    import torch

    want = torch.complex64 if precision == "single" else torch.complex128
    if not (t.is_cuda and t.is_contiguous() and t.dtype == want):
        raise ValueError(f"device output must be a contiguous CUDA {want} tensor")


def _head(tn, tree, sliced_indices, s1, slice_range, precision, mode, stats, device, out_dev,
          batch_ok=True) -> HeadVector:
    if batch_ok and _slice_batch and precision == "single" and tree.first_cut is not None:
        n_all = 1 << len(sliced_indices)
        a0, b0 = slice_range if slice_range is not None else (0, n_all)
        k = min(_slice_batch, len(sliced_indices))
        from .slice_batch import compute_head_vector_slice_batched

        # the widest aligned block that fits (rank <= 32, device memory);
        # otherwise the per-slice path below
        while k and 0 <= a0 < b0 <= n_all:
            if a0 % (1 << k) == 0 and b0 % (1 << k) == 0:
                try:
                    return compute_head_vector_slice_batched(
                        tn, tree, sliced_indices, s1, slice_range, batch_log2=k,
                        precision=precision, mode=mode, stats=stats, device=device)
                except BlockTooWide:
                    pass
                except RuntimeError as exc:
                    if "out of memory" not in str(exc):
                        raise
                    clear_cache()
            k -= 1
    s1 = normalize_s1(tn, s1)
    tn = tn.repin(s1)
    sliced_indices = list(sliced_indices)
    head_leaves, head_steps, _, _, cut = _split(tn, tree)
    head_set = set(head_leaves)
    for ix in sliced_indices:
        eps = tn.index_endpoints.get(ix, ())
        if len(eps) != 2 or any(e not in head_set for e in eps):
            raise ShapeMismatch(f"sliced index {ix} is not internal to the head")
    n_e = len(sliced_indices)
    total = 1 << n_e
    a, b = slice_range if slice_range is not None else (0, total)
    if not (0 <= a < b <= total):
        raise RangeOutOfBounds(f"range [{a},{b}) outside [0,{total})")
    if mode not in _MODES:
        raise ValueError(f"unknown reduction mode {mode!r}")
    dtype = DTYPES[precision]
    if stats is not None:
        stats.head_contractions += b - a
    if not head_leaves:
        # degenerate head (engine.py:282-283): every slice contributes ones(1)
        data = _degenerate_sum(b - a, dtype, mode)
        if out_dev is not None:
            import torch

            out_dev.copy_(torch.from_numpy(data))
            data = None
    else:
        run_steps = _exec_head_steps(tn, tree, head_leaves, head_steps, sliced_indices)
        entries = _leaf_entries(tn, head_leaves)
        prog = get_program(entries, _steps_tuples(run_steps), sliced_indices, sorted(cut),
                           precision, device, upload=False)
        if out_dev is not None and out_dev.numel() != prog.info.out_elems:
            raise ShapeMismatch(f"device output holds {out_dev.numel()} elements, "
                                f"the head vector {prog.info.out_elems}")
        if out_dev is not None:
            import torch

            torch.cuda.synchronize(out_dev.device)  # the tensor's producers (torch streams)
        data = prog.run(entries, a, b, mode, out=None if out_dev is None else out_dev.data_ptr())
        if stats is not None:
            sets = {nid: tn.nodes[nid].indices for nid in head_leaves}
            mults, _ = step_mults(sets, head_steps, frozenset(sliced_indices))
            stats.multiplications += mults * (b - a)
            stats.steps_executed += len(head_steps) * (b - a)
    return HeadVector(
        s1=s1,
        data=data,
        provenance=provenance_hash(tn, tree, s1, precision, mode, sliced_indices),
        cut_order=sorted(cut),
        n_e=n_e,
        slice_range=(a, b),
        mode=mode,
        sliced_indices=tuple(sliced_indices),
    )


def _degenerate_sum(count, dtype, mode):
    # sum of `count` scalars 1.0: exact in both modes
    return np.array([float(count)], dtype=dtype)


_tail_plan_cache: dict = {}


def tail_plan(tn, tree, cut, head_id=None):
    """Leaves + pairwise order of the head-absorbed tail network, memoised per
    topology (the order does not depend on leaf values).  The order comes
    from the native planner (``treeopt.order_network``: greedy, then exact
    subset-DP re-optimisation under the B200 time model), intermediates
    capped at 2^31 elements where the network allows."""
    _, _, tail_leaves, _, _ = _split(tn, tree)
    hid = (max(tn.nodes) + 1) if head_id is None else head_id
    key = (tuple((nid, tuple(tn.nodes[nid].indices)) for nid in tail_leaves), tuple(cut), hid)
    hit = _tail_plan_cache.get(key)
    if hit is not None:
        return tail_leaves, hid, hit
    from .treeopt import order_network

    sets = {nid: frozenset(tn.nodes[nid].indices) for nid in tail_leaves}
    sets[hid] = frozenset(cut)
    steps = order_network(sets, hid + 1, cap_log2=31)
    with _cache_lock:
        if len(_tail_plan_cache) >= 16:
            _tail_plan_cache.pop(next(iter(_tail_plan_cache)))
        _tail_plan_cache[key] = steps
    return tail_leaves, hid, steps


def compute_tail_amplitudes(tn, tree, head: HeadVector, space_cap=None, precision="double",
                            stats=None, device=None) -> AmplitudeTable:
    """All 2**n_open amplitudes of the head/tail split (engine.py:313-378)."""
    s1 = head.s1
    tn = tn.repin(s1)
    expect = provenance_hash(tn, tree, s1, precision, head.mode, head.sliced_indices)
    if expect != head.provenance:
        raise ProvenanceMismatch("head vector was produced from different inputs")
    if head.slice_range != (0, 1 << head.n_e):
        raise ProvenanceMismatch("head vector is a partial; reduce it first")
    return _tail(tn, tree, head, space_cap, precision, stats, device)


def tail_amplitudes_unchecked(tn, tree, head: HeadVector, space_cap=None, precision="single",
                              stats=None, device=None) -> AmplitudeTable:
    """Tail of a (possibly partial) head vector without the full-range check.

    The tail is linear in the head vector, so the amplitudes of a partial
    slice range are the partial amplitude sums (used for sharded runs and
    fixed-subset benchmarks)."""
    return _tail(tn.repin(head.s1), tree, head, space_cap, precision, stats, device)


def _tail(tn, tree, head, space_cap, precision, stats, device):
    _, _, tail_leaves, tail_steps, cut = _split(tn, tree)
    if sorted(cut) != list(head.cut_order):
        raise ProvenanceMismatch("cut indices differ from the head vector's")
    dtype = DTYPES[precision]
    open_qubits = sorted(tn.open_output_indices)
    n2 = len(open_qubits)
    n_c = head.n_c
    amplitudes = np.zeros(1 << n2, dtype=dtype)
    if not tail_leaves:
        amplitudes[0] = head.data.reshape(()) if head.data.size == 1 else head.data[0]
        return _make_table(tn, tree, head, amplitudes, open_qubits, precision)

    # reference-equivalent instrumentation (engine.py:348-377)
    k = 0
    if space_cap is not None:
        while n2 - k + n_c > space_cap and k < n2:
            k += 1
    if stats is not None:
        pinned = frozenset(tn.open_output_indices[q] for q in open_qubits[:k])
        sets = {nid: tn.nodes[nid].indices for nid in tail_leaves}
        mults, _ = step_mults(sets, tail_steps, pinned)
        blocks = 1 << k
        stats.tail_contractions += blocks
        stats.multiplications += blocks * (mults + (1 << (n2 - k + n_c)))
        stats.steps_executed += blocks * len(tail_steps)

    leaves, hid, steps = tail_plan(tn, tree, head.cut_order)
    entries = _leaf_entries(tn, leaves)
    entries.append((hid, list(head.cut_order), np.asarray(head.data).reshape(-1)))
    open_ids = [tn.open_output_indices[q] for q in open_qubits]
    sets = {nid: ix for nid, ix, _ in entries}
    # blocked fallback (engine.py:348-362): pin the k leading open qubits
    # (s2 MSBs) when the absorbed tail's largest intermediate exceeds
    # space_cap, or when its program does not fit in device memory; block j
    # then fills amplitudes[j << (n2 - k) : (j + 1) << (n2 - k)]
    kb = 0
    if space_cap is not None:
        while kb < n2 and step_mults(sets, steps, frozenset(open_ids[:kb]))[1] > space_cap:
            kb += 1
    while True:
        # cache keyed on topology only: the head leaf is re-uploaded when it changes
        try:
            prog = get_program(entries, steps, open_ids[:kb], open_ids[kb:], precision, device,
                               upload=False)
            break
        except RuntimeError as exc:
            if "out of memory" not in str(exc) or kb >= n2:
                raise
            clear_cache()
            kb += 1
    if kb == 0:
        amps = prog.run(entries, 0, 1, "fixed")
    else:
        amps = np.empty(1 << n2, dtype=dtype)
        w = 1 << (n2 - kb)
        with prog.lock:  # one upload of the leaves (the head vector), then every block
            prog._update_leaves(entries)
            for j in range(1 << kb):
                amps[j * w:(j + 1) * w] = prog._run_range(j, j + 1, "fixed", None)
    return _make_table(tn, tree, head, amps.astype(dtype, copy=False), open_qubits, precision)


def tail_amplitudes_to_device(tn, tree, head: HeadVector, head_dev, out,
                              precision="single", device=None) -> AmplitudeTable:
    """Head-absorbed tail of a head vector that is already in device memory
    (``head_dev``: torch CUDA tensor, 2^n_c elements of the precision's complex
    dtype); the 2^n2 amplitudes (s2 order) are written to the torch CUDA
    tensor ``out``.
    Leaf upload, head-pointer binding and run are one critical section on the
    cached program.  Returns the table's metadata with ``amplitudes=None``."""
    tn = tn.repin(head.s1)
    _, _, tail_leaves, _, cut = _split(tn, tree)
    if sorted(cut) != list(head.cut_order):
        raise ProvenanceMismatch("cut indices differ from the head vector's")
    open_qubits = sorted(tn.open_output_indices)
    if not tail_leaves:
        raise ShapeMismatch("tail_amplitudes_to_device needs a non-empty tail")
    leaves, hid, steps = tail_plan(tn, tree, head.cut_order)
    entries = _leaf_entries(tn, leaves)
    entries.append((hid, list(head.cut_order), np.zeros(1 << len(head.cut_order))))
    out_order = [tn.open_output_indices[q] for q in open_qubits]
    _check_out(head_dev, precision)
    _check_out(out, precision)
    if head_dev.numel() != 1 << len(head.cut_order) or out.numel() != 1 << len(open_qubits):
        raise ShapeMismatch("device head / amplitude tensors have the wrong size")
    prog = get_program(entries, steps, [], out_order, precision, device, upload=False)
    import torch

    torch.cuda.synchronize(out.device)
    prog.run(entries[:-1], 0, 1, "fixed", out=out.data_ptr(),
             device_leaves={len(entries) - 1: head_dev.data_ptr()})
    return _make_table(tn, tree, head, None, open_qubits, precision)


def _make_table(tn, tree, head, amplitudes, open_qubits, precision):
    csha = circuit_sha(tn)
    return AmplitudeTable(
        s1=head.s1,
        open_qubits=open_qubits,
        amplitudes=amplitudes,
        layout_ids=sorted(tn.circuit.layout.ids) if tn.circuit else
        sorted(set(tn.open_output_indices) | set(tn.fixed_output_bits)),
        circuit_sha256=csha,
        order_sha256=order_sha256(tree, tn, head.sliced_indices),
        precision=precision,
        mode=head.mode,
    )


def contract_tree(tn, tree, slice_assignment, dtype=np.complex128, stats=None, device=None):
    """Whole-tree contraction, sliced indices pinned, root axes ascending (engine.py:147-165)."""
    precision = "double" if np.dtype(dtype) == np.complex128 else "single"
    sliced = sorted(slice_assignment)
    leaves = _leaf_entries(tn, list(tree.leaves))
    steps = _steps_tuples(tree.steps)
    # root ids: leaf indices minus pinned ones, contracted pairwise
    sets = {nid: frozenset(ix) - frozenset(sliced) for nid, ix, _ in leaves}
    for (l, r, o) in steps:
        sets[o] = sets.pop(l) ^ sets.pop(r)
    if len(sets) != 1:
        raise ShapeMismatch(f"{len(sets)} results left after contraction")
    root_ids = sorted(next(iter(sets.values())))
    # indices that are not in the network at all are ignored, as np.take never sees them
    present = {i for _, ix, _ in leaves for i in ix}
    pinned = [ix for ix in sliced if ix in present]
    mask = 0
    for ix in pinned:
        mask = (mask << 1) | (int(slice_assignment[ix]) & 1)
    prog = get_program(leaves, steps, pinned, root_ids, precision, device, upload=False)
    out = prog.run(leaves, mask, mask + 1, "fixed")
    if stats is not None:
        mults, _ = step_mults({nid: ix for nid, ix, _ in leaves}, steps, frozenset(pinned))
        stats.multiplications += mults
        stats.steps_executed += len(steps)
    return out.astype(dtype, copy=False).reshape((2,) * len(root_ids))


def reduce_partials(partials) -> HeadVector:
    """Combine disjoint-range partial head vectors (engine.py:398-452)."""
    if not partials:
        raise RangeGap("no partials given")
    prov = partials[0].provenance
    n_e = partials[0].n_e
    for p in partials[1:]:
        if p.provenance != prov:
            raise ProvenanceMismatch("partials come from different runs")
        if p.n_e != n_e:
            raise ProvenanceMismatch("partials disagree on slice count")
    ordered = sorted(partials, key=lambda p: p.slice_range[0])
    pos = 0
    for p in ordered:
        a, b = p.slice_range
        if a < pos:
            raise RangeOverlap(f"range [{a},{b}) overlaps at {pos}")
        if a > pos:
            raise RangeGap(f"missing slice range [{pos},{a})")
        pos = b
    total = 1 << n_e
    if pos != total:
        raise RangeGap(f"missing slice range [{pos},{total})")

    from .device import DeviceAdder  # torch-backed device buffers
    adder = DeviceAdder(ordered[0].data.dtype, ordered[0].data.size, _default_device)

    def combine(lo, hi, items):
        if len(items) == 1 and items[0].slice_range == (lo, hi):
            return adder.upload(items[0].data)
        mid = (lo + hi) // 2
        left = [p for p in items if p.slice_range[1] <= mid]
        right = [p for p in items if p.slice_range[0] >= mid]
        if len(left) + len(right) == len(items) and left and right:
            return adder.add(combine(lo, mid, left), combine(mid, hi, right))
        acc = adder.upload(items[0].data)
        for p in items[1:]:
            acc = adder.add(acc, adder.upload(p.data))
        return acc

    data = adder.download(combine(0, total, ordered))
    return dataclasses.replace(ordered[0], data=data, slice_range=(0, total))


def flop_estimate(complexity) -> float:
    """8 FLOPs per counted multiplication (engine.py:455-458)."""
    return 8.0 * float(complexity.tc)
