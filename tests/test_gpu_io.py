"""File-based ranged partials from the GPU path (TNCUTHV1), reduced -- needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import io

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["single", "double"])
def test_gpu_partials_through_files_reduce_bit_exactly(gpu, workloads, tmp_path, precision):
    w = workloads("c1")
    full = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, precision=precision)
    paths = []
    for a in (8, 0):  # out of order, as separate workers would finish
        hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(a, a + 8),
                                     precision=precision)
        paths.append(tmp_path / f"part{a}.hv")
        io.write_head_vector(paths[-1], hv)
    red = tnb.reduce_partials([io.read_head_vector(p) for p in paths])
    assert np.array_equal(red.data, full.data)
    tab = tnb.compute_tail_amplitudes(w.tn, w.tree, red, precision=precision)
    ref = tnb.compute_tail_amplitudes(w.tn, w.tree, full, precision=precision)
    assert np.array_equal(tab.amplitudes, ref.amplitudes)
    io.write_amplitude_tsv(tmp_path / "amps.tsv", tab)
    lines = (tmp_path / "amps.tsv").read_text().splitlines()
    assert len(lines) == 2 + (1 << len(tab.open_qubits))
    assert lines[2].split("\t")[0] == tab.bitstring(0)


@pytest.mark.gpu
def test_c_abi_nccl_allreduce_single_rank(gpu):
    """tnb_allreduce_sum over a 1-rank communicator (the only NCCL shape a
    1-GPU box allows): the collective path runs and leaves the sum intact."""
    import torch

    from paper_2103_03074_b200.distributed import NcclComm

    uid = NcclComm.unique_id()
    comm = NcclComm(1, uid, 0, 0)
    x = (torch.randn(1 << 20, dtype=torch.complex64, device="cuda"))
    ref = x.clone()
    comm.allreduce_sum(x)
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    y = torch.randn(1000, dtype=torch.complex128, device="cuda")
    yr = y.clone()
    comm.allreduce_sum(y, stream=torch.cuda.current_stream())
    assert torch.equal(y, yr)
    comm.close()


def _sharded_worker(rank, world, port, out_q):
    import os
    import sys

    from conftest import ROOT

    sys.path.insert(0, ROOT)
    os.environ["LOCAL_RANK"] = str(rank)
    import torch
    import torch.distributed as dist

    from paper_2103_03074_b200 import distributed as D
    from paper_2103_03074_b200.workloads import load_workload

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = load_workload("s8")
    hv = D.sharded_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 8), mode="fixed")
    tab = D.sharded_amplitudes(w.tn, w.tree, w.sliced, None, slice_range=(0, 8), mode="fixed")
    out_q.put((rank, torch.cuda.current_device(), hv.data, hv.slice_range, tab.amplitudes))
    dist.destroy_process_group()


def test_sharded_device_path_two_ranks_one_gpu(gpu, workloads):
    """distributed.sharded_* on their default (device-resident) path, 2 ranks
    sharing the box's GPU over gloo: head -> tail -> collective never leave
    the device until the final result; fixed mode equals the 1-process
    result bit-exactly, amplitudes within fp32 rounding."""
    import socket

    import torch.multiprocessing as mp

    from conftest import rel_l2

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = workloads("s8")
    full = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 8),
                                   precision="single")
    amps = tnb.tail_amplitudes_unchecked(w.tn, w.tree, full, precision="single").amplitudes
    for rank, dev, data, rng, a in res:
        assert rng == (0, 8) and dev == 0
        assert np.array_equal(data, full.data), f"rank {rank}: fixed-mode head not bit-identical"
        e = rel_l2(a, amps)
        print(f"rank {rank}: sharded amplitudes rel L2 {e:.2e}")
        assert e < 1e-5


def test_device_resident_api_validates_and_matches_host_api(gpu, workloads):
    """engine.head_vector_to_device / tail_amplitudes_to_device: same numbers
    as the host API; wrong dtype / size / host tensors are rejected."""
    import torch

    from conftest import measured, rel_l2
    from paper_2103_03074_b200 import engine as E

    w = workloads("s8")
    hv = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 4),
                                 precision="single")
    tab = tnb.tail_amplitudes_unchecked(w.tn, w.tree, hv, precision="single")
    dev = torch.device("cuda", 0)
    head = torch.empty(hv.data.size, dtype=torch.complex64, device=dev)
    meta = E.head_vector_to_device(w.tn, w.tree, w.sliced, None, head, slice_range=(0, 4),
                                   precision="single")
    assert meta.data is None and meta.slice_range == (0, 4) and meta.provenance == hv.provenance
    assert np.array_equal(head.cpu().numpy(), hv.data)
    amps = torch.empty(tab.amplitudes.size, dtype=torch.complex64, device=dev)
    t2 = E.tail_amplitudes_to_device(w.tn, w.tree, meta, head, amps, precision="single")
    assert t2.amplitudes is None and t2.open_qubits == tab.open_qubits
    assert measured(rel_l2(amps.cpu().numpy(), tab.amplitudes)) < 1e-6
    with pytest.raises(ValueError):
        E.head_vector_to_device(w.tn, w.tree, w.sliced, None, head.to(torch.complex128),
                                slice_range=(0, 4), precision="single")
    with pytest.raises(ValueError):
        E.head_vector_to_device(w.tn, w.tree, w.sliced, None, head.cpu(), slice_range=(0, 4),
                                precision="single")
    with pytest.raises(tnb.ShapeMismatch):
        E.head_vector_to_device(w.tn, w.tree, w.sliced, None, head[:-1], slice_range=(0, 4),
                                precision="single")


@pytest.mark.parametrize("mode", ["fixed", "free"])
def test_threaded_multi_device_head_vector(gpu, workloads, mode):
    """distributed.threaded_head_vector: one thread per device (here 4
    threads sharing the box's GPU), aligned ranges, reduce_partials' tree --
    fixed mode bit-identical to one call over the whole range."""
    from conftest import measured, rel_l2
    from paper_2103_03074_b200.distributed import threaded_head_vector

    w = workloads("s8")
    full = tnb.compute_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 16),
                                   precision="single", mode=mode)
    got = threaded_head_vector(w.tn, w.tree, w.sliced, None, slice_range=(0, 16),
                               precision="single", mode=mode, devices=[0, 0, 0, 0])
    assert got.slice_range == (0, 16) and got.provenance == full.provenance
    if mode == "fixed":
        assert np.array_equal(got.data, full.data)
    else:
        assert measured(rel_l2(got.data, full.data)) < 1e-6
