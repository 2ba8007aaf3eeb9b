"""Benchmark: slices/s and contraction TFLOP/s on the m=20 Sycamore-53 plan.

Workload (BASELINE.json configs[3], SURVEY 8 "C4"): Sycamore-layout 53-qubit
m=20 circuit (synthetic gates, seed 0), 20 open qubits -> a 2^20 correlated
bitstring batch, reference plan (seed 0 / restarts 16 / target space 2^30,
n_e = 53 sliced edges, n_c = 21 cut indices), frozen under tests/golden/c4.
A *step* = a batch of `--slices` head slices per GPU: sliced-leaf gather,
413 pairwise contractions per slice (tcgen05 GEMMs for the big ones),
on-device fixed-mode slice sum, then the head-absorbed sparse-state tail
over the 2^20 bitstrings and (N > 1) one NCCL all-reduce of the amplitude
vector.  Ranks own disjoint aligned slice ranges of a fixed subset
(weak scaling).

    python bench.py [--gpus N --steps K --warmup W]      # this executor
    python bench.py --impl reference ...                 # reference CPU path

Without a launcher, ``--gpus N`` spawns N rank processes (torchrun's env);
under torchrun it uses the launcher's ranks.  Beside the headline the line
carries optional legs (batched s1, co-optimised plan, re-ordered tree,
batched slices, double precision, cross-slice reuse), each reported
separately, and the reference engine's own CPU time (``cpu_baseline``).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

HOST_CORES = len(os.sched_getaffinity(0))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(HOST_CORES))

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "slices/sec & contraction TFLOP/s, Sycamore-53 m=20 correlated batch, 1-8 GPU"
WORKLOAD = "c4"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]), float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                try:
                    pw.append(float(r[3]))
                except ValueError:
                    pass
                for k, nm in enumerate(names):
                    if r[4 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": float(np.median(pw)) if pw else None}


# ---------------------------------------------------------------------------
# TNB_* variables a benchmark of record may carry: launch plumbing only.  Every
# other TNB_* knob (tile/pacing/fusion overrides, debug prints, the GEMM's
# promotion chunk) changes the executed schedule, so the bench refuses to run
# with one set unless --allow-knobs marks the line as a diagnostic run.
_BENCH_ENV_OK = {"TNB_SHARE_DEVICE", "TNB_DIST_BACKEND", "TNB_REF_BUDGET_S", "TNB_PLAN_THREADS",
                 "TNB_BENCH_FAIL_LEG", "TNB_BENCH_FAIL_LEG_RANK", "TNB_BENCH_FAIL_RANK",
                 "TNB_BENCH_PROFILE_E2E"}


def diagnostic_knobs():
    return sorted(k for k in os.environ if k.startswith("TNB_") and k not in _BENCH_ENV_OK)


def refuse_diagnostics(allow=False):
    knobs = diagnostic_knobs()
    if knobs and not allow:
        raise SystemExit(f"bench: refusing to run with executor knobs set ({', '.join(knobs)}); "
                         "unset them or pass --allow-knobs (the line is then marked diagnostic)")
    return knobs


def spawn_ranks(n: int, argv) -> int:
    """``python bench.py --gpus N`` without a launcher: start N rank processes
    of this script exactly as torchrun would (RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_ADDR=127.0.0.1 / MASTER_PORT in the env, one device per rank) and
    return the worst exit code.  Rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *argv], env=env))
    # like torchrun: a rank that fails takes the others down (they would
    # otherwise wait in their next collective forever)
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            rc = max(rc, code)
            if code != 0:
                for q in live:
                    q.terminate()
                for q in live:
                    try:
                        q.wait(timeout=30)
                    except subprocess.TimeoutExpired:
                        q.kill()
                live = []
                break
        time.sleep(0.2)
    return rc


def setup_dist(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    # test hook: TNB_SHARE_DEVICE=1 puts every rank on device 0 (gloo), so the
    # multi-rank choreography can be exercised on a single-GPU box
    if os.environ.get("TNB_SHARE_DEVICE") == "1":
        local = 0
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_

        if args.impl == "ours" and torch.cuda.is_available():
            torch.cuda.set_device(local)
        backend = os.environ.get("TNB_DIST_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        dist_.init_process_group(backend)
        dist = dist_
    return world, rank, local, dist


def rank_inventory(dist, local):
    """Which device every rank drives (PCI bus id): evidence that N ranks
    ran on N distinct GPUs, plus the communicator's size and backend."""
    import torch

    me = {"rank": int(os.environ.get("RANK", "0")), "device": local}
    if torch.cuda.is_available():
        p = torch.cuda.get_device_properties(local)
        me["pci_bus_id"] = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}"
        me["name"] = p.name
    ranks = [me]
    comm = {"backend": None, "size": 1}
    if dist is not None:
        ranks = [None] * dist.get_world_size()
        dist.all_gather_object(ranks, me)
        comm = {"backend": dist.get_backend(), "size": dist.get_world_size()}
        if comm["backend"] == "nccl":
            try:
                v = torch.cuda.nccl.version()
                comm["nccl_version"] = ".".join(map(str, v)) if isinstance(v, tuple) else str(v)
            except Exception:  # noqa: BLE001 - informational only
                comm["nccl_version"] = None
    active = len({r.get("pci_bus_id", r["device"]) for r in ranks})
    return ranks, active, comm


def barrier(dist, local):
    import torch

    if dist is not None:
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize(local)


def traffic_from_profile():
    """DRAM bytes per GEMM launch from the committed ncu capture of this bench
    (scripts/make_traffic_json.py -> profiles/r2/gemm_traffic.json), else null."""
    path = os.path.join(ROOT, "profiles", "r2", "gemm_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        return {"traffic": t["dram_bytes_per_launch"], "traffic_unit": "bytes/launch (DRAM read+write)",
                "traffic_algorithmic": t.get("algorithmic_bytes_per_launch"),
                "traffic_over_algorithmic": t.get("dram_over_algorithmic"),
                "traffic_source": t["source"]}
    except Exception:
        return {"traffic": None}


def cpu_baseline(w, budget_s):
    """One real reference slice (kind "reference"); the sampler of
    oracle/cpu_sample.py only when the reference is not importable."""
    line = reference_cpu_baseline(w, budget_s)
    if "unavailable" not in line:
        return line
    from oracle.cpu_sample import time_head_slice

    est, wall, sample = time_head_slice(w.tn, w.tree, w.sliced, precision="single")
    flops = 8.0 * w.tc_per_slice
    return {"value": 1.0 / est, "unit": "slices/s", "cores": HOST_CORES, "kind": "port",
            "sample": "EXTRAPOLATED sampler (reference unavailable: " + line["unavailable"] + "): " + sample,
            "est_s_per_slice": est, "tflops": flops / est / 1e12}


def _run_leg(name, fn, dist=None, dev=None):
    """An optional bench leg.  ``fn`` does only rank-local work (no
    collectives) and returns ``(result, local, finalize)``: ``local`` maps
    the leg's timings to this rank's values, ``finalize(maxed)`` fills the
    result from their max over ranks.  The wrapper makes ONE all-reduce per
    leg with a failure flag in it, so a leg that fails on one rank (e.g.
    device memory on a shared box) cannot leave the other ranks waiting in a
    collective: every rank marks it unavailable and the bench continues."""
    keys, failed, res, local, fin = [], 0, None, {}, None
    try:
        if os.environ.get("TNB_BENCH_FAIL_LEG") == name and (
                os.environ.get("TNB_BENCH_FAIL_LEG_RANK") in (None, os.environ.get("RANK", "0"))):
            raise RuntimeError("injected failure")  # test hook
        res, local, fin = fn()
        keys = sorted(local)
    except Exception as exc:  # noqa: BLE001
        failed = 1
        print(f"[bench] leg {name} failed: {exc!r}", file=sys.stderr, flush=True)
        res = {"unavailable": f"{type(exc).__name__}: {str(exc)[:200]}"}
        try:
            from paper_2103_03074_b200 import engine as _E

            _E.clear_cache()
        except Exception:  # noqa: BLE001
            pass
    maxed = dict(local)
    if dist is not None:
        import torch

        # the key set is the leg's own (identical on every rank that got that far);
        # a failed rank contributes the flag and zeros
        n = torch.tensor([len(keys)], device=dev, dtype=torch.int64)
        dist.all_reduce(n, op=dist.ReduceOp.MAX)
        width = int(n.item())
        vals = [float(failed)] + [float(local[k]) for k in keys] + [0.0] * (width - len(keys))
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if t[0].item() > 0 and not failed:
            res = {"unavailable": "failed on another rank (see its stderr)"}
            failed = 1
        maxed = {k: float(t[1 + i].item()) for i, k in enumerate(keys)}
    if failed or res is None:
        return res
    if fin is not None:
        fin(maxed)
    return res


def run_dry(args):
    """The multi-rank plumbing of run_ours without kernels (CPU tests): the
    rendezvous, the per-rank aligned slice ranges, one all-reduce of an
    amplitude-sized vector and the max-over-ranks timing."""
    import torch

    os.environ.setdefault("TNB_DIST_BACKEND", "gloo")
    world, rank, local, dist = setup_dist(args)
    ranks, active, comm = rank_inventory(dist, local)
    total = (args.warmup + args.steps) * args.slices
    mine = (rank * total, (rank + 1) * total)
    if os.environ.get("TNB_BENCH_FAIL_RANK") == str(rank):  # test hook: a rank dies before the collective
        raise SystemExit(f"rank {rank}: injected failure")
    amps = torch.full((1 << 10,), float(rank + 1), dtype=torch.float32)
    t0 = time.perf_counter()
    if dist is not None:
        dist.all_reduce(amps)
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3])
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        spans = [None] * world
        dist.all_gather_object(spans, mine)
    else:
        spans = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks, "gpus_active": active,
                          "communicator": comm, "slice_ranges": spans,
                          "allreduce_sum": float(amps[0]), "max_ms": float(ms[0])}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_ours(args):
    import torch

    import paper_2103_03074_b200 as tnb
    from paper_2103_03074_b200 import engine as E
    from paper_2103_03074_b200.planner import split

    world, rank, local, dist = setup_dist(args)
    if world > 1:  # host planning threads per rank (the plan legs run treeopt on every rank)
        os.environ.setdefault("TNB_PLAN_THREADS", str(max(1, HOST_CORES // world)))
    torch.cuda.set_device(local)
    tnb.set_device(local)
    ranks, gpus_active, comm = rank_inventory(dist, local)
    w = tnb.load_workload(args.workload)
    S = args.slices
    total_slices = (args.warmup + args.steps) * S
    base = rank * total_slices  # aligned disjoint per-rank range of the fixed subset
    tn, tree = w.tn, w.tree
    hl, hs, tl, ts, cut = split(tn, tree)
    head = E.head_program(tn, tree, w.sliced, "single", device=local)
    # timed region: GEMM launches + range totals only (events around the
    # hundreds of small kernels would add their issue cost to the measured
    # time); the per-class breakdown comes from one extra, separate step
    head.set_timing(2)
    n_c = len(cut)
    opens = sorted(tn.open_output_indices)
    n2 = len(opens)
    leaves, hid, tsteps = E.tail_plan(tn, tree, sorted(cut))
    entries = E._leaf_entries(tn, leaves) + [(hid, sorted(cut), np.zeros(1 << n_c))]
    tail = E.get_program(entries, tsteps, [], [tn.open_output_indices[q] for q in opens], "single",
                         device=local)
    tail.set_timing(2)
    dev = torch.device("cuda", local)
    hvec = torch.empty(1 << n_c, dtype=torch.complex64, device=dev)
    amps = torch.empty(1 << n2, dtype=torch.complex64, device=dev)
    amps_total = torch.zeros(1 << n2, dtype=torch.complex64, device=dev)

    def step(s, accumulate=True):
        a = base + s * S
        head.run_range(a, a + S, "fixed", out=hvec.data_ptr())
        tail.set_leaf_device(len(entries) - 1, hvec.data_ptr())
        tail.run_range(0, 1, "fixed", out=amps.data_ptr())
        th, tt = head.timing(), tail.timing()
        ms = th["total_ms"] + tt["total_ms"]
        if dist is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dist.all_reduce(amps.view(torch.float32))
            e1.record()
            e1.synchronize()
            ms += e0.elapsed_time(e1)
        if accumulate:
            amps_total.add_(amps)
        return ms, th, tt

    for s in range(args.warmup):
        step(s)
    barrier(dist, local)
    dev_ms = 0.0
    gemm_ms = gemm_flops = 0.0
    launches = gemm_launches = 0
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for s in range(args.warmup, args.warmup + args.steps):
            ms, th, tt = step(s)
            dev_ms += ms
            gemm_ms += th["gemm_ms"] + tt["gemm_ms"]
            gemm_flops += th["gemm_flops"] + tt["gemm_flops"]
            launches += th["launches"] + tt["launches"]
            gemm_launches += th["gemm_launches"] + tt["gemm_launches"]
        barrier(dist, local)
    wall_ms = (time.perf_counter() - t0) * 1e3
    # per-class breakdown (not timed as the headline): one more step with
    # events around every kernel class
    head.set_timing(1)
    tail.set_timing(1)
    _, bh, bt = step(args.warmup + args.steps, accumulate=False)
    breakdown = {k: bh[k] + bt[k] for k in ("convert_ms", "simt_ms", "other_ms")}
    breakdown_total = bh["total_ms"] + bt["total_ms"]
    breakdown_gemm = bh["gemm_ms"] + bt["gemm_ms"]
    head.set_timing(2)
    tail.set_timing(2)
    # max over ranks of the device time
    t_max = dev_ms
    if dist is not None:
        tt_ = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        t_max = float(tt_.item())

    # ---- e2e: the public API with host buffers (H2D of every leaf, D2H of results)
    e2e = None
    if not args.no_e2e:
        hprog = head
        # one untimed pass through the public API first (the device leg had W
        # warm-up steps; this one pages in the pinned result buffers)
        a = base + (args.warmup - 1) * S
        hprog._leaf_data = [None] * hprog.n_leaves
        hv = tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a, a + S),
                                     precision="single", device=local)
        tnb.tail_amplitudes_unchecked(tn, tree, hv, precision="single", device=local)
        barrier(dist, local)
        h2d = d2h = 0
        e2e_dev_ms = 0.0  # device time of the same calls (program events)
        prof = None
        if os.environ.get("TNB_BENCH_PROFILE_E2E"):
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        e_t0 = time.perf_counter()
        for s in range(args.steps):
            a = base + (args.warmup + s) * S
            hprog._leaf_data = [None] * hprog.n_leaves  # inputs arrive from the host every call
            hv = tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a, a + S),
                                         precision="single", device=local)
            e2e_dev_ms += hprog.timing()["total_ms"]
            tab = tnb.tail_amplitudes_unchecked(tn, tree, hv, precision="single", device=local)
            e2e_dev_ms += tail.timing()["total_ms"]  # the engine's cached tail program
            h2d += sum(8 * (1 << len(tn.nodes[n].indices)) for n in hl)
            h2d += 8 * (1 << n_c)  # head vector into the tail program
            d2h += hv.data.nbytes + tab.amplitudes.nbytes
        barrier(dist, local)
        e_ms = (time.perf_counter() - e_t0) * 1e3
        if prof is not None:
            import pstats

            prof.disable()
            pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(18)
        if dist is not None:
            tt_ = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
            e_ms = float(tt_.item())
        e2e = {"value": world * args.steps * S / (e_ms / 1e3), "unit": "slices/s",
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "ms_per_step": e_ms / args.steps,
               "device_ms_per_step": e2e_dev_ms / args.steps}

    # ---- optional: batched closed-bit assignments --
    # 2^b s1 values in one head pass over the same slices; reported beside
    # the headline as assignment-slices/s (a bigger correlated batch)
    def sync():
        torch.cuda.synchronize(local)

    def _leg_batched():
        if args.batch_s1 <= 0:
            return None, {}, None
        from paper_2103_03074_b200.batched import cheapest_batch_qubits, compute_head_vectors_batched

        qs, ratio = cheapest_batch_qubits(tn, tree, w.sliced, args.batch_s1)
        closed = sorted(tn.fixed_output_bits)
        s1_list = []
        for v in range(1 << len(qs)):
            s = dict(tn.fixed_output_bits)
            for i, q in enumerate(qs):
                s[q] = (v >> (len(qs) - 1 - i)) & 1
            s1_list.append("".join(str(s[q]) for q in closed))
        a = base
        compute_head_vectors_batched(tn, tree, w.sliced, s1_list, slice_range=(a, a + S),
                                     precision="single", device=local)  # compile + warm
        sync()
        b_t0 = time.perf_counter()
        for s_ in range(args.steps):
            a = base + s_ * S
            compute_head_vectors_batched(tn, tree, w.sliced, s1_list, slice_range=(a, a + S),
                                         precision="single", device=local)
        sync()
        b_ms = (time.perf_counter() - b_t0) * 1e3 / args.steps
        batched = {"assignments": len(s1_list), "qubits": qs, "analytic_cost_ratio": ratio,
                   "bitstrings_per_pass": len(s1_list) << len(tn.open_output_indices),
                   "note": "head vectors of 2^b closed-bit assignments from one contraction with "
                           "those qubits' output legs open (paper_2103_03074_b200.batched; equal to "
                           "per-s1 runs, tests/test_batched.py); wall time incl. host copies"}
        E.clear_cache()

        def fin(m):
            batched["ms_per_step"] = m["b_ms"]
            batched["assignment_slices_per_s"] = world * S * len(s1_list) / (m["b_ms"] / 1e3)
        return batched, {"b_ms": b_ms}, fin

    batched = _run_leg("batched", _leg_batched, dist, dev)

    # ---- optional: the co-optimised plan of the same network:
    # same head leaves / cut / head vector, head tree + sliced set from
    # treeopt.select_slices_b200 (frozen in tests/golden/<workload>_opt31_b200,
    # else _opt_b200, else _opt).
    # Reported beside the headline: slices of a different plan are a
    # different unit; the comparable figure is the time for ALL slices.
    def _leg_opt_plan():
        opt_name = next((args.workload + sfx for sfx in ("_opt31_b200", "_opt_b200", "_opt")
                         if os.path.isdir(os.path.join(ROOT, "tests", "golden", args.workload + sfx))), None)
        if not (args.opt_plan and opt_name is not None):
            return None, {}, None
        wo = tnb.load_workload(opt_name)
        op = E.head_program(wo.tn, wo.tree, wo.sliced, "single", device=local)
        op.set_timing(2)
        So = args.opt_slices
        ob = rank * (args.warmup + args.steps) * So
        for s_ in range(args.warmup):
            op.run_range(ob + s_ * So, ob + (s_ + 1) * So, "fixed", out=hvec.data_ptr())
        sync()
        o_ms = o_gemm_ms = o_gemm_flops = 0.0
        o_launches = 0
        for s_ in range(args.warmup, args.warmup + args.steps):
            op.run_range(ob + s_ * So, ob + (s_ + 1) * So, "fixed", out=hvec.data_ptr())
            t = op.timing()
            o_ms += t["total_ms"]
            o_gemm_ms += t["gemm_ms"]
            o_gemm_flops += t["gemm_flops"]
            o_launches += t["launches"]
        opt_plan = {"workload": opt_name, "n_e": wo.n_e,
                    "target_space": wo.target_space, "flops_per_slice": 8.0 * wo.tc_per_slice,
                    "gemm_tflops": o_gemm_flops / (o_gemm_ms / 1e3) / 1e12 if o_gemm_ms else 0.0,
                    "slices_per_step_per_gpu": So, "launches_per_step": o_launches / args.steps,
                    "planner": wo.doc.get("planner", {}).get("tool"),
                    "note": "device time of the co-optimised plan's head slices (same network, head "
                            "leaves, cut and head vector as the reference plan; tests/test_gpu_treeopt.py "
                            "pins its results to the reference engine run on that plan)"}
        del op
        E.clear_cache()
        # the co-optimised plan's slices in 2^k blocks (slice_batch.py, rank <= 32);
        # the block width comes from a time-budgeted host search, so ranks may
        # differ: each runs its own, the line reports the range
        from paper_2103_03074_b200 import slice_batch as SB

        for ko in (3, 2, 1):
            try:
                SB.batched_plan(wo.tn, wo.tree, wo.sliced, ko, max_rank=32)
                break
            except (tnb.ShapeMismatch, tnb.TncutError, ValueError):
                ko = 0
        bo_ms = 0.0
        if ko:
            bo = SB.batched_program(wo.tn, wo.tree, wo.sliced, ko, "single", local, max_rank=32)
            bo.set_timing(2)
            ob2 = (1 << (wo.n_e - ko)) // 2 + rank * (args.warmup + args.steps)
            for s_ in range(args.warmup):
                bo.run_range(ob2 + s_, ob2 + s_ + 1, "fixed", out=hvec.data_ptr())
            sync()
            for s_ in range(args.warmup, args.warmup + args.steps):
                bo.run_range(ob2 + s_, ob2 + s_ + 1, "fixed", out=hvec.data_ptr())
                bo_ms += bo.timing()["total_ms"]
            del bo
            E.clear_cache()

        def fin(m):
            sps = world * args.steps * So / (m["o_ms"] / 1e3)
            opt_plan.update(slices_per_s=sps, contraction_tflops=sps * 8.0 * wo.tc_per_slice / 1e12,
                            all_slices_head_s_log2=wo.n_e - math.log2(sps))
            k_lo, k_hi = int(-m["neg_ko"]), int(m["ko"])
            if k_lo > 0 and m["bo_ms"] > 0:
                bsps = world * args.steps * (1 << k_lo) / (m["bo_ms"] / 1e3)
                opt_plan["batched"] = {"batch_log2": k_lo, "slices_per_s": bsps,
                                       "all_slices_head_s_log2": wo.n_e - math.log2(bsps)}
                if k_hi != k_lo:
                    opt_plan["batched"]["note"] = f"block width differed across ranks ({k_lo}..{k_hi})"
        return opt_plan, {"o_ms": o_ms, "bo_ms": bo_ms, "ko": float(ko), "neg_ko": -float(ko)}, fin

    opt_plan = _run_leg("opt_plan", _leg_opt_plan, dist, dev)

    # ---- optional: the SAME slices (reference sliced set, same masks, same
    # partial head vectors) through a re-ordered head tree
    # (treeopt keep_slices; tests/golden/<workload>_reordered).  Reported
    # beside the headline, which executes the reference tree as given.
    def _leg_reordered():
        ro_name = args.workload + "_reordered"
        if not (args.reordered and os.path.isdir(os.path.join(ROOT, "tests", "golden", ro_name))):
            return None, {}, None
        wr = tnb.load_workload(ro_name)
        assert wr.sliced == w.sliced
        # the re-ordered tree with its small steps clustered, as set_reorder runs it
        from paper_2103_03074_b200.planner import cluster_small_steps

        _hl, _hs, _, _, _cut = E._split(wr.tn, wr.tree)
        _steps = cluster_small_steps({n: wr.tn.nodes[n].indices for n in _hl}, _hs,
                                     frozenset(wr.sliced))
        rp = E.get_program(E._leaf_entries(wr.tn, _hl), E._steps_tuples(_steps), list(wr.sliced),
                           sorted(_cut), "single", local)
        rp.set_timing(2)
        Sr = args.reordered_slices
        rb = rank * (args.warmup + args.steps) * Sr
        for s_ in range(args.warmup):
            rp.run_range(rb + s_ * Sr, rb + (s_ + 1) * Sr, "fixed", out=hvec.data_ptr())
        sync()
        r_ms = r_gemm_ms = r_gemm_flops = 0.0
        r_launches = 0
        for s_ in range(args.warmup, args.warmup + args.steps):
            rp.run_range(rb + s_ * Sr, rb + (s_ + 1) * Sr, "fixed", out=hvec.data_ptr())
            t = rp.timing()
            r_ms += t["total_ms"]
            r_gemm_ms += t["gemm_ms"]
            r_gemm_flops += t["gemm_flops"]
            r_launches += t["launches"]
        reordered = {"workload": ro_name,
                     "executed_flops_per_slice": 8.0 * wr.tc_per_slice,
                     "gemm_tflops": r_gemm_flops / (r_gemm_ms / 1e3) / 1e12 if r_gemm_ms else 0.0,
                     "slices_per_step_per_gpu": Sr, "launches_per_step": r_launches / args.steps,
                     "note": "the reference plan's own slices (same sliced set and masks, same partial "
                             "head vectors: tests/test_gpu_treeopt.py) with the head tree re-ordered by "
                             "treeopt (keep_slices, exact subtree DP + B200 polish); executed FLOPs "
                             "are the re-ordered tree's"}
        del rp
        E.clear_cache()
        # the same through the public API (set_reorder; host buffers, leaves
        # H2D and the head vector D2H every call)
        tnb.set_reorder(True)
        try:
            a0 = base + total_slices  # slices beyond the headline subset
            tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a0, a0 + Sr),
                                    precision="single", device=local)  # plan + compile
            sync()
            e_t0 = time.perf_counter()
            for s_ in range(args.steps):
                a = a0 + (s_ + 1) * Sr
                tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a, a + Sr),
                                        precision="single", device=local)
            sync()
            re_ms = (time.perf_counter() - e_t0) * 1e3
        finally:
            tnb.set_reorder(False)
        E.clear_cache()

        def fin(m):
            rsps = world * args.steps * Sr / (m["r_ms"] / 1e3)
            reordered.update(slices_per_s=rsps, executed_tflops=rsps * 8.0 * wr.tc_per_slice / 1e12,
                             e2e_api_slices_per_s=world * args.steps * Sr / (m["re_ms"] / 1e3))
        return reordered, {"r_ms": r_ms, "re_ms": re_ms}, fin

    reordered = _run_leg("reordered", _leg_reordered, dist, dev)

    # ---- optional: batched slices (slice_batch.py): 2^k aligned slices of the
    # SAME plan per contraction (the k lowest-mask-bit sliced indices
    # un-sliced), head tree re-ordered for the reduced sliced set
    def _leg_batched_slices():
        if args.batch_slices <= 0:
            return None, {}, None
        from paper_2103_03074_b200 import slice_batch as SB

        kb = args.batch_slices
        while True:  # the largest k <= --batch-slices whose intermediates fit rank 32
            try:
                steps_b, reduced_b, sc_b = SB.batched_plan(tn, tree, w.sliced, kb)
                break
            except tnb.ShapeMismatch:
                kb -= 1
                if kb == 0:
                    raise
        bp = SB.batched_program(tn, tree, w.sliced, kb, "single", local)
        bp.set_timing(2)
        Bb = 4  # blocks per step
        # blocks beyond the headline subset, disjoint per rank
        bb = ((world * total_slices) >> kb) + 1 + rank * (args.warmup + args.steps) * Bb
        for s_ in range(args.warmup):
            bp.run_range(bb + s_ * Bb, bb + (s_ + 1) * Bb, "fixed", out=hvec.data_ptr())
        sync()
        b_ms = b_gemm_ms = b_gemm_flops = 0.0
        for s_ in range(args.warmup, args.warmup + args.steps):
            bp.run_range(bb + s_ * Bb, bb + (s_ + 1) * Bb, "fixed", out=hvec.data_ptr())
            t = bp.timing()
            b_ms += t["total_ms"]
            b_gemm_ms += t["gemm_ms"]
            b_gemm_flops += t["gemm_flops"]
        from paper_2103_03074_b200.planner import step_mults

        mb, _ = step_mults({n: tn.nodes[n].indices for n in hl}, steps_b, frozenset(reduced_b))
        batched_slices = {"batch_log2": kb, "max_rank": sc_b,
                          "executed_flops_per_slice": 8.0 * mb / (1 << kb),
                          "gemm_tflops": b_gemm_flops / (b_gemm_ms / 1e3) / 1e12 if b_gemm_ms else 0.0,
                          "speedup_vs_headline": None,
                          "note": "the reference plan's slices, 2^k aligned slices per contraction "
                                  "(lowest-mask-bit sliced indices un-sliced, tree re-ordered; "
                                  "tests/test_gpu_slice_batch.py); executed FLOPs are the batched tree's"}
        del bp
        E.clear_cache()
        # the same through the public API (set_slice_batch; host buffers)
        tnb.set_slice_batch(kb)
        try:
            a0 = (bb + (args.warmup + args.steps) * Bb) << kb
            tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a0, a0 + (Bb << kb)),
                                    precision="single", device=local)  # plan + compile
            sync()
            e_t0 = time.perf_counter()
            for s_ in range(args.steps):
                a = a0 + ((s_ + 1) * Bb << kb)
                tnb.compute_head_vector(tn, tree, w.sliced, None, slice_range=(a, a + (Bb << kb)),
                                        precision="single", device=local)
            sync()
            be_ms = (time.perf_counter() - e_t0) * 1e3
        finally:
            tnb.set_slice_batch(0)
        E.clear_cache()

        def fin(m):
            sps_b = world * args.steps * Bb * (1 << kb) / (m["b_ms"] / 1e3)
            batched_slices.update(slices_per_s=sps_b,
                                  executed_tflops=sps_b * 8.0 * mb / (1 << kb) / 1e12,
                                  e2e_api_slices_per_s=world * args.steps * (Bb << kb) / (m["be_ms"] / 1e3))
            if int(-m["neg_kb"]) != int(m["kb"]):
                batched_slices["note_ranks"] = (f"block width differed across ranks "
                                                f"({int(-m['neg_kb'])}..{int(m['kb'])})")
        return batched_slices, {"b_ms": b_ms, "be_ms": be_ms, "kb": float(kb), "neg_kb": -float(kb)}, fin

    batched_slices = _run_leg("batched_slices", _leg_batched_slices, dist, dev)

    # ---- optional: double precision (the reference's default, engine.py:248):
    # the same slices on the fp64 path (DMMA / FMA; tcgen05 has no fp64 kind)
    def _leg_double():
        if not args.double:
            return None, {}, None
        E.clear_cache()
        dp = E.head_program(tn, tree, w.sliced, "double", device=local)
        dp.set_timing(2)
        d0 = base
        dp.run_range(d0, d0 + 1, "fixed")  # compile + warm
        sync()
        d_ms = 0.0
        for s_ in range(args.double):
            dp.run_range(d0 + 1 + s_, d0 + 2 + s_, "fixed")
            d_ms += dp.timing()["total_ms"]
        del dp
        E.clear_cache()
        res = {"slices_per_gpu": args.double,
               "note": "precision='double' (complex128; the reference's default) on the fp64 path "
                       "(DMMA mma.sync m8n8k4 for the big steps, FMA for the rest), same slices and "
                       "tree as the headline; device time"}

        def fin(m):
            sps = world * args.double / (m["d_ms"] / 1e3)
            res.update(slices_per_s=sps, contraction_tflops=sps * 8.0 * w.tc_per_slice / 1e12)
        return res, {"d_ms": d_ms}, fin

    double_leg = _run_leg("double", _leg_double, dist, dev)

    # ---- optional: cross-slice reuse (TNB_FLAG_REUSE_SLICES) -- reported beside the
    # headline, NOT as it: it skips re-computing results whose mask bits did not change
    def _leg_reuse():
        if not args.reuse:
            return None, {}, None
        from paper_2103_03074_b200 import _lib as L

        # e.g. the dedicated cache buffers exceeding HBM -> the leg is unavailable
        rprog = E.head_program(tn, tree, w.sliced, "single", device=local,
                               flags=L.TNB_FLAG_REUSE_SLICES)
        rprog.set_timing(2)
        rbase = base + total_slices  # fresh slices beyond the headline subset
        for s in range(args.warmup):
            rprog.run_range(rbase + s * S, rbase + (s + 1) * S, "fixed", out=hvec.data_ptr())
        sync()
        r_ms = r_gemm_ms = r_gemm_flops = 0.0
        r_reused = 0
        for s in range(args.warmup, args.warmup + args.steps):
            rprog.run_range(rbase + s * S, rbase + (s + 1) * S, "fixed", out=hvec.data_ptr())
            t = rprog.timing()
            r_ms += t["total_ms"]
            r_gemm_ms += t["gemm_ms"]
            r_gemm_flops += t["gemm_flops"]
            r_reused += t["steps_reused"]
        res = {"unit": "slices/s",
               "executed_gemm_tflops": r_gemm_flops / (r_gemm_ms / 1e3) / 1e12 if r_gemm_ms else 0,
               "executed_flop_fraction": r_gemm_flops / (args.steps * S * 8.0 * w.tc_per_slice),
               "steps_reused": r_reused, "cache_bytes": int(rprog.info.reuse_bytes),
               "note": "head slices with TNB_FLAG_REUSE_SLICES: steps whose mask bits did not "
                       "change between consecutive slices are not recomputed (results "
                       "bit-identical, tests/test_gpu_parity.py); tail excluded"}
        del rprog
        E.clear_cache()

        def fin(m):
            res["value"] = world * args.steps * S / (m["r_ms"] / 1e3)
        return res, {"r_ms": r_ms}, fin

    if args.reuse:
        import gc

        E.clear_cache()
        del head, tail, step  # the closure holds the programs too
        gc.collect()
    reuse = _run_leg("reuse", _leg_reuse, dist, dev)

    if rank != 0:
        return
    burst, sustained, hbm, src = peaks()
    slices = world * args.steps * S
    value = slices / (t_max / 1e3)
    flops_slice = 8.0 * w.tc_per_slice
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else 0.0
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "slices/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c64 (fp16x3-split tcgen05, fp32 accumulate)",
        "data": "synthetic (Sycamore-layout random gates, seed 0; reference plan frozen in tests/golden/c4)",
        "config": {"workload": f"{args.workload.upper()}: Sycamore-53 m=20, 2^{n2} correlated bitstrings, "
                               f"target space 2^{w.target_space}, n_e={w.n_e}, n_c={n_c}, "
                               "fixed subset of slices",
                   "slices_per_step_per_gpu": S, "slice_subset": [0, world * total_slices],
                   "l2": "inputs larger than L2 (intermediates up to 8 GiB)",
                   "parallelism": f"slice-range dp{world}"},
        "contraction_tflops": value * flops_slice / 1e12,
        "flops_per_slice": flops_slice,
        "roofline": {
            "bound": "tensor", "kernel": "gemm_f16x3 (tcgen05)",
            "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
            "frac": achieved / sustained,
            "peak_kind": (f"{src} bf16 dense sustained " +
                          ("(MEASURED_PEAKS.json)" if src == "measured"
                           else "(B200_PROFILING.md fallback: MEASURED_PEAKS.json absent)")),
            "achieved_is": "algorithmic complex FLOPs (8 per complex multiply-add) per GEMM launch / event time",
            "tensor_tflops_executed": 3.0 * achieved,
            "tensor_frac": 3.0 * achieved / sustained,
            # the complex-algorithmic ceiling of the chosen
            # decomposition is P/g' -- here one real GEMM on the 2x2 real form
            # (= 4M) run as 3 fp16 split products, i.e. peak/3
            "method_ceiling": sustained / 3.0,
            "frac_of_method_ceiling": achieved / (sustained / 3.0),
            **traffic_from_profile(),
        },
        "gpu_launches": launches,
        "gpus_active": gpus_active,
        "ranks": ranks,
        "communicator": comm,
        "device_ms_per_step": {"total": dev_ms / args.steps, "gemm": gemm_ms / args.steps,
                               "non_gemm": (dev_ms - gemm_ms) / args.steps},
        "breakdown_step_ms": {"note": "one extra step after the timed region with CUDA events "
                                      "around every kernel class (their issue cost included)",
                              "total": breakdown_total, "gemm": breakdown_gemm, **breakdown,
                              "gaps": breakdown_total - breakdown_gemm - sum(breakdown.values())},
        "gemm_launches": gemm_launches,
        "wall_ms_per_step": wall_ms / args.steps,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cross_slice_reuse": reuse,
        "batched_s1": batched,
        "co_optimised_plan": opt_plan,
        "reordered_same_slices": reordered,
        "batched_slices": batched_slices,
        "double_precision": double_leg,
        # linear XEB (analytics.py:46-58) of the synthetic partial amplitudes
        # accumulated over every bench step (the fixed slice subset)
        "xeb_partial_subset": float((2.0 ** 53 / amps_total.numel())
                                    * float((amps_total.abs().double() ** 2).sum()) - 1.0),
    }
    if reordered and "unavailable" not in reordered:
        reordered["speedup_vs_headline"] = reordered["slices_per_s"] / value
    if batched_slices and "unavailable" not in batched_slices:
        batched_slices["speedup_vs_headline"] = batched_slices["slices_per_s"] / value
    if opt_plan and "unavailable" not in opt_plan:
        # time for ALL 2^n_e head slices, reference plan vs co-optimised plan
        ref_log2 = w.n_e - math.log2(value)
        opt_plan["reference_plan_all_slices_head_s_log2"] = ref_log2
        opt_plan["all_slices_speedup_log2"] = ref_log2 - opt_plan["all_slices_head_s_log2"]
        if opt_plan.get("batched"):
            opt_plan["batched"]["all_slices_speedup_log2"] = ref_log2 - opt_plan["batched"]["all_slices_head_s_log2"]
    if getattr(args, "knobs", None):
        line["diagnostic_knobs"] = {k: os.environ[k] for k in args.knobs}
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(w, args.ref_budget_s)
    print(json.dumps(line), flush=True)


REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")  # pip --target install of the reference


def import_reference():
    """The UNMODIFIED reference package ``tncut`` from baseline/_ref (pip
    --target install, travels to the GPU box); /root/reference/pkg/src in
    the build container.  None when neither is importable."""
    for path in (REF_INSTALL, "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tncut")) and path not in sys.path:
            sys.path.insert(0, path)
            break
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tnb")
    try:
        import tncut  # noqa: F401
        from tncut import engine  # noqa: F401
    except Exception as exc:  # noqa: BLE001
        return None, f"{type(exc).__name__}: {exc}"
    return tncut, None


def reference_workload(name):
    """Network + plan through the reference's OWN builders: parse_circuit
    (circuit.py), build_network (network.py), doc_to_tree (ordering.py:670-722)
    on the frozen circuit/order files of tests/golden/<name>."""
    from tncut import ordering
    from tncut.circuit import parse_circuit
    from tncut.network import build_network

    d = os.path.join(ROOT, "tests", "golden", name)
    with open(os.path.join(d, "circuit.qsim")) as fh:
        circ = parse_circuit(fh.read(), "qsim_text")
    with open(os.path.join(d, "order.json")) as fh:
        doc = json.load(fh)
    if circ.sha256() != doc["circuit_sha256"]:
        raise RuntimeError(f"{name}: circuit sha mismatch")
    opens = doc["open_qubits"]
    tn = build_network(circ, set(opens), {q: 0 for q in circ.layout.ids if q not in set(opens)})
    return tn, ordering.doc_to_tree(doc), list(doc["slices"]), doc


def time_reference_slices(name, first, max_slices, budget_s):
    """Wall time of the reference's own ``compute_head_vector(tn, tree,
    sliced, None, slice_range=(a, a+1), precision="single", mode="fixed")``
    (engine.py:242-310), one real slice per call, until ``max_slices`` calls
    or until the next call would overrun ``budget_s``.  No extrapolation:
    returns the per-slice wall times actually measured."""
    from tncut import engine

    tn, tree, sliced, doc = reference_workload(name)
    times = []
    t_all = time.perf_counter()
    while len(times) < max_slices:
        spent = time.perf_counter() - t_all
        if times and spent + max(times) > budget_s:
            break
        a = first + len(times)
        t0 = time.perf_counter()
        engine.compute_head_vector(tn, tree, sliced, None, slice_range=(a, a + 1),
                                   precision="single", mode="fixed")
        times.append(time.perf_counter() - t0)
    return times


def reference_cpu_baseline(w, budget_s):
    """cpu_baseline leg of our arm: real reference slices (kind "reference")."""
    ref, why = import_reference()
    if ref is None:
        return {"unavailable": f"reference not importable: {why}"}
    times = time_reference_slices(WORKLOAD, 0, 1, budget_s)
    s = float(sum(times))
    return {"value": len(times) / s, "unit": "slices/s", "cores": HOST_CORES, "kind": "reference",
            "sample": f"{len(times)} full C4 head slice(s) [0,{len(times)}) through the unmodified "
                      f"reference engine (baseline/_ref tncut.engine.compute_head_vector, "
                      f"precision=single, mode=fixed), OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}; "
                      f"{s:.1f} s measured, no extrapolation",
            "s_per_slice": s / len(times), "tflops": len(times) * 8.0 * w.tc_per_slice / s / 1e12}


def run_reference(args):
    """--impl reference: the reference's CPU engine on this box's host cores.

    A C4 slice is ~70-110 s of OpenBLAS on 16 cores, so K full slices do not
    fit the driver's step budget.  Each timed step is ONE real reference
    slice; steps run until K or until --ref-budget-s would be exceeded, and
    the line reports the number actually timed (``steps``) beside the
    requested K.  Warm-up steps are C1 head slices through the same engine
    (imports, numba JIT, OpenBLAS thread pool), not timed."""
    world = int(os.environ.get("WORLD_SIZE", "1")) if "WORLD_SIZE" in os.environ else args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    base = {"metric": METRIC, "impl": "reference"}
    ref, why = import_reference()
    if ref is None:
        print(json.dumps({**base, "unavailable": f"reference not importable from baseline/_ref: {why}"}),
              flush=True)
        return
    from tncut import engine

    from paper_2103_03074_b200.workloads import load_workload

    w = load_workload(args.workload)  # tc_per_slice / n_e bookkeeping only
    tn1, tree1, sl1, _ = reference_workload("c1")
    for s in range(args.warmup):
        engine.compute_head_vector(tn1, tree1, sl1, None, slice_range=(s % 16, s % 16 + 1),
                                   precision="single", mode="fixed")
    t0 = time.perf_counter()
    times = time_reference_slices(args.workload, 0, args.steps, args.ref_budget_s)
    wall = time.perf_counter() - t0
    total = float(sum(times))
    v = len(times) / total
    sample = (f"{len(times)} full {args.workload.upper()} head slices [0,{len(times)}) of the reference "
              f"plan, one compute_head_vector(slice_range=(a,a+1), precision='single', mode='fixed') "
              f"call each (unmodified tncut from baseline/_ref), OPENBLAS_NUM_THREADS="
              f"{os.environ.get('OPENBLAS_NUM_THREADS')}; no extrapolation")
    line = {**base, "value": v, "unit": "slices/s", "n_gpus": world, "steps": len(times),
            "requested_steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64 (numpy/OpenBLAS cgemm)",
            "data": "synthetic (Sycamore-layout random gates, seed 0; reference plan frozen in tests/golden/c4)",
            "config": {"workload": f"{args.workload.upper()}: Sycamore-53 m=20, 2^20 correlated bitstrings, "
                                   f"target space 2^{w.target_space}, n_e={w.n_e}",
                       "parallelism": "host CPU (rank 0 only)"},
            "contraction_tflops": v * 8.0 * w.tc_per_slice / 1e12,
            "per_slice_s": times,
            "steps_note": (f"each step is one full reference slice; {len(times)} of the requested "
                           f"{args.steps} fit the {args.ref_budget_s:.0f} s budget"
                           if len(times) < args.steps else "all requested steps timed"),
            "warmup_note": "warm-up steps are C1 head slices through the same reference engine",
            "cpu_baseline": {"value": v, "unit": "slices/s", "cores": HOST_CORES, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "timed_wall_s": wall}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--slices", type=int, default=2, help="head slices per step per GPU")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/rendezvous/collective plumbing only (gloo, no kernels): CPU tests")
    ap.add_argument("--allow-knobs", action="store_true",
                    help="run with TNB_* executor knobs set (the line is marked diagnostic)")
    ap.add_argument("--ref-budget-s", type=float, default=float(os.environ.get("TNB_REF_BUDGET_S", "420")),
                    help="wall budget of the reference arm's timed slices (each ~62-69 s at C4 on 16 cores)")
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--reuse", type=int, default=1, help="also time TNB_FLAG_REUSE_SLICES (reported separately)")
    ap.add_argument("--opt-plan", type=int, default=1,
                    help="also time the co-optimised plan <workload>_opt (reported separately)")
    ap.add_argument("--opt-slices", type=int, default=4, help="co-optimised plan slices per step per GPU")
    ap.add_argument("--reordered", type=int, default=1,
                    help="also time the same slices through the re-ordered tree <workload>_reordered")
    ap.add_argument("--reordered-slices", type=int, default=16)
    ap.add_argument("--batch-slices", type=int, default=4,
                    help="also time 2^k-slice blocks per contraction (slice_batch.py; 0 = off)")
    ap.add_argument("--double", type=int, default=1,
                    help="also time N head slices in double precision (reported separately; 0 = off)")
    ap.add_argument("--batch-s1", type=int, default=4,
                    help="also time 2^b closed-bit assignments per head pass (reported separately)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if os.environ.get("TNB_SHARE_DEVICE") != "1" and not args.dry_run:
            import torch

            n_dev = torch.cuda.device_count()
            if n_dev < args.gpus:
                raise SystemExit(f"bench: --gpus {args.gpus} but only {n_dev} visible CUDA device(s)")
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        args.knobs = refuse_diagnostics(args.allow_knobs)
        run_ours(args)
        import torch.distributed as dist_

        if dist_.is_available() and dist_.is_initialized():
            dist_.barrier()  # rank 0 has printed; leave together
            dist_.destroy_process_group()


if __name__ == "__main__":
    main()
