"""Multi-process slice sharding logic with gloo, world_size 2 (CPU).

The per-rank partial is computed by the oracle (injected), so this checks
the range partitioning, the collective choreography and the combine order
of paper_2103_03074_b200.distributed -- the device kernels are covered by
the GPU tests.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, rel_l2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, out_q):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import engine_np as O
    from paper_2103_03074_b200 import distributed as D
    from paper_2103_03074_b200.types import AmplitudeTable, HeadVector
    from paper_2103_03074_b200.workloads import load_workload

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = load_workload("s8")

    def head_partial(lo, hi):
        data = O.head_vector(w.tn, w.tree, w.sliced, (lo, hi), "single", mode)
        hv = HeadVector(s1={}, data=data, provenance="p", cut_order=[], n_e=w.n_e,
                        slice_range=(lo, hi), mode=mode)
        return torch.from_numpy(data), hv

    hv = D.sharded_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 8), mode=mode,
                               partial_fn=head_partial)

    def amp_partial(lo, hi):
        data = O.head_vector(w.tn, w.tree, w.sliced, (lo, hi), "single", mode)
        amps = O.tail_absorbed(w.tn, w.tree, data, precision="single")
        tab = AmplitudeTable(s1={}, open_qubits=[], amplitudes=amps, layout_ids=[],
                             circuit_sha256="", order_sha256="", precision="single", mode=mode)
        return torch.from_numpy(amps), tab

    tab = D.sharded_amplitudes(w.tn, w.tree, w.sliced, None, slice_range=(0, 8), mode=mode,
                               partial_fn=amp_partial)
    out_q.put((rank, hv.data, hv.slice_range, tab.amplitudes))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fixed", "free"])
def test_two_rank_sharding_matches_single_process(workloads, mode):
    from oracle import engine_np as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = workloads("s8")
    full = O.head_vector(w.tn, w.tree, w.sliced, (0, 8), "single", mode)
    amps = O.tail_absorbed(w.tn, w.tree, full, precision="single")
    for rank, data, rng, a in res:
        assert rng == (0, 8)
        if mode == "fixed":
            # aligned power-of-two partials recombine bit-exactly (engine.py:398-405)
            assert np.array_equal(data, full)
        else:
            assert rel_l2(data, full) < 1e-6
        assert rel_l2(a, amps) < 1e-5   # linear tail: sum of partial amplitudes


def test_aligned_ranges():
    from paper_2103_03074_b200.distributed import aligned_ranges, tree_combine

    assert aligned_ranges(0, 16, 4) == [(0, 4), (4, 8), (8, 12), (12, 16)]
    assert aligned_ranges(8, 16, 2) == [(8, 12), (12, 16)]
    r = aligned_ranges(0, 10, 3)
    assert r[0][0] == 0 and r[-1][1] == 10 and all(a < b for a, b in r)
    assert tree_combine([1, 2, 3, 4], lambda x, y: f"({x}+{y})") == "((1+2)+(3+4))"
    assert tree_combine([1, 2, 3], lambda x, y: f"({x}+{y})") == "((1+2)+3)"
