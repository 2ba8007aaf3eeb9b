"""bench.py's launcher: ``--gpus N`` without torchrun spawns N ranks
(RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* like torchrun) and rank 0 prints one
line with the communicator size and the device of every rank."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra, timeout):
    env = {k: v for k, v in os.environ.items() if not k.startswith("TNB_")}
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_gpus_flag_spawns_ranks_dry_run():
    line = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1", "--slices", "2"],
                {"TNB_SHARE_DEVICE": "1"}, 180)
    assert line["n_gpus"] == 2
    assert line["communicator"] == {"backend": "gloo", "size": 2}
    assert [r["rank"] for r in line["ranks"]] == [0, 1]
    assert line["slice_ranges"] == [[0, 6], [6, 12]]  # disjoint per-rank ranges
    assert line["allreduce_sum"] == 3.0


def test_failed_rank_takes_the_others_down():
    """A rank that dies before a collective ends the job with a non-zero
    exit instead of leaving the other ranks waiting forever."""
    env = {k: v for k, v in os.environ.items() if not k.startswith("TNB_")}
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env.update(TNB_SHARE_DEVICE="1", TNB_BENCH_FAIL_RANK="1")
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run", "--steps", "1"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "injected failure" in r.stderr


def test_bench_refuses_executor_knobs():
    env = {k: v for k, v in os.environ.items() if not k.startswith("TNB_")}
    env["TNB_CHUNK_KB"] = "0"
    r = subprocess.run([sys.executable, BENCH, "--steps", "1"], capture_output=True, text=True,
                       timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "refusing" in r.stderr


def test_more_gpus_than_devices_fails():
    import torch

    if torch.cuda.device_count() >= 64:
        pytest.skip("box has 64 GPUs")
    env = {k: v for k, v in os.environ.items() if not k.startswith("TNB_")}
    r = subprocess.run([sys.executable, BENCH, "--gpus", "64", "--steps", "1"], capture_output=True,
                       text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "visible CUDA device" in r.stderr


@pytest.mark.gpu
def test_bench_two_ranks_share_one_gpu(gpu):
    """The full bench step on 2 ranks (gloo, both on device 0: the 1-GPU box
    can not host 2 NCCL ranks): head -> tail -> all-reduce per rank, max
    over ranks, rank 0's line."""
    line = _run(["--gpus", "2", "--steps", "1", "--warmup", "1", "--slices", "1", "--no-cpu",
                 "--no-e2e", "--reuse", "0", "--opt-plan", "0", "--reordered", "0",
                 "--batch-slices", "0", "--batch-s1", "0", "--double", "0"],
                {"TNB_SHARE_DEVICE": "1", "TNB_DIST_BACKEND": "gloo"}, 900)
    assert line["n_gpus"] == 2 and line["communicator"]["size"] == 2
    assert line["gpus_active"] == 1 and line["value"] > 0
    assert line["gpu_launches"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_all_legs_c2(gpu):
    """Every optional leg on 2 ranks (gloo, shared GPU) on the smaller C2
    plan: the legs' collectives (plan-choice agreement, max-over-ranks
    times) line up on both ranks and rank 0 prints one complete line."""
    line = _run(["--gpus", "2", "--workload", "c2", "--steps", "1", "--warmup", "1", "--slices", "1",
                 "--no-cpu", "--reuse", "1", "--opt-plan", "1", "--opt-slices", "1", "--reordered", "1",
                 "--reordered-slices", "2", "--batch-slices", "2", "--batch-s1", "2", "--double", "1"],
                {"TNB_SHARE_DEVICE": "1", "TNB_DIST_BACKEND": "gloo"}, 1500)
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["value"] > 0
    for leg in ("batched_s1", "co_optimised_plan", "batched_slices", "double_precision",
                "cross_slice_reuse"):
        assert line[leg] is not None and "unavailable" not in line[leg], (leg, line[leg])


def test_reference_arm_times_real_reference_slices():
    """--impl reference: the unmodified reference engine (baseline/_ref or the
    reference tree) on real slices, no extrapolation (C1 here: fast)."""
    import importlib.util

    if not (os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "tncut"))
            or os.path.isdir("/root/reference/pkg/src/tncut")):
        pytest.skip("reference package not present")
    if importlib.util.find_spec("numba") is None:
        pytest.skip("reference dependencies missing")
    line = _run(["--impl", "reference", "--workload", "c1", "--steps", "3", "--warmup", "1"], {}, 300)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["steps"] == 3 and line["requested_steps"] == 3 and len(line["per_slice_s"]) == 3
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert abs(line["value"] - 3 / sum(line["per_slice_s"])) < 1e-9 * line["value"]


def test_reference_arm_budget_caps_the_timed_slices(monkeypatch):
    """Slices stop once the next one would overrun the budget (the driver's
    step budget cannot hold K full C4 slices); the line says so."""
    import importlib.util

    if importlib.util.find_spec("numba") is None or not (
            os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "tncut"))
            or os.path.isdir("/root/reference/pkg/src/tncut")):
        pytest.skip("reference package not present")
    line = _run(["--impl", "reference", "--workload", "c1", "--steps", "50", "--warmup", "0",
                 "--ref-budget-s", "0"], {}, 300)
    assert line["steps"] == 1 and line["requested_steps"] == 50
    assert "fit" in line["steps_note"]


@pytest.mark.gpu
def test_bench_leg_failing_on_one_rank_does_not_hang(gpu):
    """A leg that fails on rank 1 only (injected; e.g. device memory) is
    reported unavailable on every rank and the other legs still run: the
    legs' timings meet in one all-reduce per leg with a failure flag."""
    line = _run(["--gpus", "2", "--workload", "c2", "--steps", "1", "--warmup", "1", "--slices", "1",
                 "--no-cpu", "--no-e2e", "--reuse", "0", "--opt-plan", "0", "--reordered", "0",
                 "--batch-slices", "2", "--batch-s1", "0", "--double", "1"],
                {"TNB_SHARE_DEVICE": "1", "TNB_DIST_BACKEND": "gloo",
                 "TNB_BENCH_FAIL_LEG": "batched_slices", "TNB_BENCH_FAIL_LEG_RANK": "1"}, 900)
    assert "unavailable" in line["batched_slices"]
    assert line["double_precision"]["slices_per_s"] > 0
