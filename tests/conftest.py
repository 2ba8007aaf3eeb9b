"""Shared test helpers.

``-m "not gpu"``: oracle vs reference golden vectors, host logic, C-ABI
load/exports, multi-process (gloo) sharding logic.  ``-m gpu``: parity of
the CUDA path (through the C-ABI) against the oracle and the goldens.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU and libtnb.so")


# measured parity errors, printed at the end of the run (GPU logs show margins)
PARITY = []


def parity_report(tag, **errs):
    """Record measured errors of one comparison (printed in the summary)."""
    PARITY.append((tag, {k: float(v) for k, v in errs.items()}))
    print(f"[parity] {tag}: " + ", ".join(f"{k}={v:.3e}" for k, v in errs.items()))


def measured(err, what="rel_l2"):
    """Record an error measured inside the current test and return it."""
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0].split("::")[-1]
    PARITY.append((test, {what: float(err)}))
    return err


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not PARITY:
        return
    tr = terminalreporter
    tr.section("measured parity errors (each test asserts its own bound; north_star: rel L2 1e-4, XEB abs 1e-3)")
    for tag, errs in PARITY:
        tr.write_line(f"{tag}: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    worst = {}
    for tag, errs in PARITY:
        for k, v in errs.items():
            if k.startswith("control"):  # negative controls (expected to be large) are listed only
                continue
            kind = "xeb" if "xeb" in k else "rel"
            if v > worst.get(kind, (-1, ""))[0]:
                worst[kind] = (v, tag)
    tr.write_line("parity worst: " + "; ".join(f"{k} {v:.2e} ({t})" for k, (v, t) in sorted(worst.items()))
                  + f"; {len(PARITY)} comparisons")


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128).reshape(-1)
    b = np.asarray(b, dtype=np.complex128).reshape(-1)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def golden(name):
    path = os.path.join(GOLDEN, name, "golden.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden vectors for {name} not generated")
    return np.load(path)


def reference_available() -> bool:
    return os.path.isdir(REF_SRC)


def import_reference():
    """The reference package (only in the build container, never on the GPU box)."""
    if not reference_available():
        pytest.skip("reference package not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import tncut  # noqa: F401

    return tncut


@pytest.fixture(scope="session")
def workloads():
    from paper_2103_03074_b200.workloads import load_workload

    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_workload(name)
        return cache[name]

    return get


@pytest.fixture(scope="session")
def gpu():
    """Skip unless a device is visible; fail loudly if the library is missing."""
    from paper_2103_03074_b200 import _lib

    lib = _lib.load()  # raises if libtnb.so was not built
    if _lib.device_count() == 0:
        pytest.skip("no CUDA device")
    return lib
