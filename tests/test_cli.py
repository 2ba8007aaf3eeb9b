"""The reference CLI (tncut) driven through paper_2103_03074_b200.cli: the
engine and analytics names inside tncut.cli / tncut.pipeline are rebound to
this executor (CPU: binding only; GPU: a full `tncut run` + `reduce`
round trip against the reference's own output)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, measured

REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")  # pip --target install of the reference


def _tncut():
    """tncut from /root/reference (build container) or baseline/_ref (GPU box)."""
    for path in ("/root/reference/pkg/src", REF_INSTALL):
        if os.path.isdir(os.path.join(path, "tncut")) and path not in sys.path:
            sys.path.insert(0, path)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        import tncut  # noqa: F401
    except Exception:
        pytest.skip("reference package not importable")


def test_bind_rebinds_engine_and_analytics_names():
    _tncut()
    import tncut.cli as cli
    import tncut.pipeline as pipeline

    from paper_2103_03074_b200 import analytics, cli as ours, engine

    prev = ours.bind()
    try:
        assert cli.compute_head_vector is engine.compute_head_vector
        assert cli.compute_tail_amplitudes is engine.compute_tail_amplitudes
        assert cli.reduce_partials is engine.reduce_partials
        assert pipeline.compute_head_vector is engine.compute_head_vector
        assert cli.xeb is analytics.xeb
        from paper_2103_03074_b200 import io as ours_io

        assert cli.write_amplitude_tsv is ours_io.write_amplitude_tsv
    finally:
        ours.unbind(prev)
    assert cli.compute_head_vector is not engine.compute_head_vector


@pytest.mark.gpu
def test_tncut_run_and_reduce_on_the_executor(gpu, tmp_path):
    """`tncut run` (full range and two partials + `tncut reduce`) on the C1
    plan through the executor; amplitudes match the reference's own run."""
    _tncut()
    import tncut.cli as cli

    from paper_2103_03074_b200 import cli as ours

    circ = os.path.join(GOLDEN, "c1", "circuit.qsim")
    order = os.path.join(GOLDEN, "c1", "order.json")

    def table(path):
        rows = [l.split("\t") for l in open(path)
                if l.strip() and not l.startswith("#") and not l.startswith("bitstring")]
        return {r[0]: complex(float(r[1]), float(r[2])) for r in rows if len(r) >= 3}

    # the reference itself (unbound)
    ref_out = tmp_path / "ref.tsv"
    with pytest.raises(SystemExit) as e:
        cli.main(args=["run", circ, order, "--precision", "double", "-o", str(ref_out)])
    assert e.value.code in (0, None)
    ref = table(ref_out)

    for precision, tol in (("double", 1e-10), ("single", 1e-4)):
        out = tmp_path / f"ours_{precision}.tsv"
        assert ours.main(["run", circ, order, "--precision", precision, "-o", str(out)]) == 0
        got = table(out)
        assert got.keys() == ref.keys()
        a = np.array([got[k] for k in ref]); b = np.array([ref[k] for k in ref])
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < tol, precision

    # `run --threads 4` (cli.py:367-380): 4 concurrent ranges through the
    # shared cached program, threads bound to devices round-robin
    out = tmp_path / "ours_threads.tsv"
    assert ours.main(["run", circ, order, "--precision", "single", "--threads", "4",
                      "-o", str(out)]) == 0
    got = table(out)
    a = np.array([got[k] for k in ref]); b = np.array([ref[k] for k in ref])
    assert measured(np.linalg.norm(a - b) / np.linalg.norm(b)) < 1e-4

    # partial ranges written by the executor, reduced by the reference's `reduce`
    import json
    n_e = len(json.load(open(order)).get("slices", []))
    if n_e >= 1:
        half = 1 << (n_e - 1)
        parts = []
        for a, b in ((0, half), (half, 2 * half)):
            p = tmp_path / f"part_{a}.hv"
            assert ours.main(["run", circ, order, "--slices", f"{a}..{b}", "-o", str(p)]) == 0
            parts.append(str(p))
        red = tmp_path / "reduced.tsv"
        assert ours.main(["reduce", *parts, "--circuit", circ, "--order", order, "-o", str(red)]) == 0
        got = table(red)
        a = np.array([got[k] for k in ref]); b = np.array([ref[k] for k in ref])
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-10


def test_tncut_slice_with_the_co_optimiser(tmp_path, monkeypatch):
    """`tncut slice` (cli.py:253-303) with select_slices rebound to the plan
    co-optimiser (TNB_CLI_SLICER=b200): a valid reference order document
    whose total head work is below the reference slicer's (CPU only)."""
    _tncut()
    import json
    import math

    import tncut.cli as cli

    from paper_2103_03074_b200 import cli as ours

    circ = os.path.join(GOLDEN, "s8", "circuit.qsim")
    order = os.path.join(GOLDEN, "s8", "order.json")
    out_ref, out_b200 = str(tmp_path / "ref.json"), str(tmp_path / "b200.json")
    args = ["slice", circ, order, "--target-space", "18", "-o"]
    with pytest.raises(SystemExit) as e:
        cli.main(args=args + [out_ref], standalone_mode=True)
    assert e.value.code in (0, None)
    monkeypatch.setenv("TNB_CLI_SLICER", "b200")
    assert ours.main(args + [out_b200]) == 0
    assert cli.select_slices is not ours.b200_select_slices  # unbound again
    ref, b200 = json.load(open(out_ref)), json.load(open(out_b200))
    tot = lambda d: math.log2(d["subtask"]["tc"]) + d["subtask"]["n_e"]  # noqa: E731
    assert b200["subtask"]["sc_log2"] <= 18
    assert tot(b200) < tot(ref)
