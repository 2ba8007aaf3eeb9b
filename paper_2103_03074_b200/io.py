"""On-disk formats of the reference engine, restated.

* ``write_head_vector`` / ``read_head_vector``: the ``TNCUTHV1`` partial
  head-vector format (engine.py:539-597), so ranged GPU partials join the
  reference's file-based multi-node flow (``tncut run --slices`` +
  ``tncut reduce``, cli.py:358-365, 417-441) byte-for-byte.
* ``write_amplitude_tsv``: the ``tncut-amplitudes/1`` table (engine.py:464-479),
  vectorised -- the reference builds 2^20-2^21 bitstrings row by row in
  Python; here the bitstring column is produced with numpy bit arithmetic.
  Output is byte-identical to the reference writer (tests/test_io.py).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import ProvenanceMismatch, ShapeMismatch
from .types import HeadVector

_HV_MAGIC = b"TNCUTHV1"
TSV_SCHEMA = "tncut-amplitudes/1"


def write_head_vector(path, head) -> None:
    """TNCUTHV1 writer (engine.py:539-560)."""
    dtype_code = 0 if head.data.dtype == np.complex128 else 1
    with open(path, "wb") as fh:
        fh.write(_HV_MAGIC)
        fh.write(struct.pack("<IB3x", 1, dtype_code))
        fh.write(head.provenance.encode("ascii"))
        fh.write(struct.pack("<II", head.n_c, head.n_e))
        fh.write(struct.pack("<QQ", *head.slice_range))
        fh.write(head.mode.encode("ascii")[:8].ljust(8, b"\0"))
        fh.write(np.asarray(head.cut_order, dtype="<u8").tobytes())
        fh.write(np.asarray(head.sliced_indices, dtype="<u8").tobytes())
        s1_items = sorted(head.s1.items())
        fh.write(struct.pack("<I", len(s1_items)))
        for q, bit in s1_items:
            fh.write(struct.pack("<QB", q, bit))
        fh.write(np.ascontiguousarray(head.data).tobytes())


def read_head_vector(path) -> HeadVector:
    """TNCUTHV1 reader (engine.py:563-597)."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != _HV_MAGIC:
            raise ProvenanceMismatch(f"not a head-vector file (magic {magic!r})")
        version, dtype_code = struct.unpack("<IB3x", fh.read(8))
        if version != 1:
            raise ProvenanceMismatch(f"unsupported head-vector version {version}")
        provenance = fh.read(64).decode("ascii")
        n_c, n_e = struct.unpack("<II", fh.read(8))
        a, b = struct.unpack("<QQ", fh.read(16))
        mode = fh.read(8).rstrip(b"\0").decode("ascii")
        cut = np.frombuffer(fh.read(8 * n_c), dtype="<u8").astype(int).tolist()
        sl = np.frombuffer(fh.read(8 * n_e), dtype="<u8").astype(int).tolist()
        (n_s1,) = struct.unpack("<I", fh.read(4))
        s1 = {}
        for _ in range(n_s1):
            q, bit = struct.unpack("<QB", fh.read(9))
            s1[q] = bit
        dtype = np.complex128 if dtype_code == 0 else np.complex64
        data = np.frombuffer(fh.read(), dtype=dtype).copy()
        if data.size != 1 << n_c:
            raise ShapeMismatch(f"payload holds {data.size} entries, expected {1 << n_c}")
    return HeadVector(s1=s1, data=data, provenance=provenance, cut_order=cut, n_e=n_e,
                      slice_range=(a, b), mode=mode, sliced_indices=tuple(sl))


def bitstrings(table) -> np.ndarray:
    """All row bitstrings of an AmplitudeTable (AmplitudeTable.bitstring, engine.py:83-92)."""
    n2 = len(table.open_qubits)
    layout = sorted(table.layout_ids)
    rows = np.arange(1 << n2, dtype=np.int64)
    cols = np.empty((rows.size, len(layout)), dtype=np.uint8)
    pos = {q: i for i, q in enumerate(table.open_qubits)}
    for c, q in enumerate(layout):
        if q in pos:
            cols[:, c] = (rows >> (n2 - 1 - pos[q])) & 1
        else:
            cols[:, c] = table.s1[q]
    cols += ord("0")
    return cols.view(f"S{len(layout)}").reshape(-1)


_iolib = None


def _io_lib():
    global _iolib
    if _iolib is None:
        import ctypes as C

        from .build import IO_LIB

        if not os.path.exists(IO_LIB):
            raise RuntimeError(f"{IO_LIB} not built (python -m paper_2103_03074_b200.build)")
        lib = C.CDLL(IO_LIB)
        lib.tnbio_row_cap.restype = C.c_int64
        lib.tnbio_row_cap.argtypes = [C.c_int32]
        lib.tnbio_format_rows.restype = C.c_int64
        lib.tnbio_format_rows.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64,
                                          C.c_void_p, C.c_int64, C.c_int32]
        _iolib = lib
    return _iolib


ROWS_PER_CHUNK = 1 << 16


def write_amplitude_tsv(path, table, threads: int = 0) -> None:
    """``tncut-amplitudes/1`` TSV (engine.py:464-479), byte-identical to the
    reference writer: bitstrings vectorised in numpy, the three number
    columns formatted by libtnbio (csrc/tsv_format.cpp) on all host threads,
    2^16 rows per chunk."""
    amps = np.asarray(table.amplitudes)
    single = amps.dtype == np.complex64
    if not single:
        amps = amps.astype(np.complex128, copy=False)
    amps = np.ascontiguousarray(amps).reshape(-1)
    s1_str = "".join(str(table.s1[q]) for q in sorted(table.s1)) or "-"
    opens = ",".join(str(q) for q in table.open_qubits) or "-"
    header = (f"# {TSV_SCHEMA} circuit_sha256={table.circuit_sha256} "
              f"order_sha256={table.order_sha256} s1={s1_str} "
              f"open_qubits={opens} n={len(table.layout_ids)} "
              f"precision={table.precision} reduction={table.mode}\n"
              "bitstring\tamp_re\tamp_im\tprobability\n")
    bits = np.ascontiguousarray(bitstrings(table))
    nb = bits.dtype.itemsize
    lib = _io_lib()
    n = amps.size
    cap = min(n, ROWS_PER_CHUNK) * lib.tnbio_row_cap(nb)
    buf = np.empty(max(cap, 1), dtype=np.uint8)
    with open(path, "wb") as fh:
        fh.write(header.encode())
        for lo in range(0, n, ROWS_PER_CHUNK):
            hi = min(n, lo + ROWS_PER_CHUNK)
            got = lib.tnbio_format_rows(bits[lo:hi].ctypes.data, nb, amps[lo:hi].ctypes.data,
                                        1 if single else 0, hi - lo, buf.ctypes.data, cap, threads)
            if got < 0:
                raise RuntimeError("tnbio_format_rows: buffer too small")
            fh.write(memoryview(buf)[:got])
