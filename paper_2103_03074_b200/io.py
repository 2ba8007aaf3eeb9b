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


def _fmt17g(x: np.ndarray) -> list:
    """Python's f'{v:.17g}' for a float array (exactly what the reference prints)."""
    return [f"{v:.17g}" for v in x.tolist()]


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


def write_amplitude_tsv(path, table) -> None:
    """``tncut-amplitudes/1`` TSV (engine.py:464-479), vectorised bitstrings."""
    amps = np.asarray(table.amplitudes)
    s1_str = "".join(str(table.s1[q]) for q in sorted(table.s1)) or "-"
    opens = ",".join(str(q) for q in table.open_qubits) or "-"
    header = (f"# {TSV_SCHEMA} circuit_sha256={table.circuit_sha256} "
              f"order_sha256={table.order_sha256} s1={s1_str} "
              f"open_qubits={opens} n={len(table.layout_ids)} "
              f"precision={table.precision} reduction={table.mode}\n"
              "bitstring\tamp_re\tamp_im\tprobability\n")
    # rows() yields complex(amp) and float(abs(amp) ** 2) with numpy SCALAR
    # arithmetic (engine.py:94-96); numpy's scalar abs/pow differ from the
    # array ufuncs in the last bit, so the probability column keeps the scalar path
    c128 = amps.astype(np.complex128)
    re = _fmt17g(c128.real)
    im = _fmt17g(c128.imag)
    pr = [f"{float(abs(v) ** 2):.17g}" for v in amps]
    bits = bitstrings(table)
    with open(path, "w", newline="\n") as fh:
        fh.write(header)
        fh.writelines(f"{b.decode()}\t{r}\t{i}\t{p}\n" for b, r, i, p in zip(bits, re, im, pr))
