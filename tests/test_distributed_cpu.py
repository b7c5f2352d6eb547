"""Host-side multi-GPU logic on CPU: shard ranges and the final gather (gloo, world_size 2)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2112_03444_b200.distributed import gather_to_rank0, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 1024, 8192, 1001):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard_range(total, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(8192, 3, 8) == (3072, 4096)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    # per-rank "results": instance ids encoded in values, complex x, int status
    x = torch.arange(lo, hi, dtype=torch.float64).repeat_interleave(3).reshape(-1, 3).to(torch.complex128) * (1 + 1j)
    st = torch.arange(lo, hi, dtype=torch.int32)
    out = gather_to_rank0([x, st])
    if rank == 0:
        q.put((out[0].numpy(), out[1].numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 7])
def test_gather_to_rank0_gloo(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    x, st = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert list(st) == list(range(total))
    assert x.shape == (total, 3)
    assert (x[:, 0].real == torch.arange(total).numpy()).all()


def _bench_worker(rank, world, port, total, q):
    """bench.py's per-rank path on CPU: instance block from bench.instance_range (strong scaling,
    uneven total), the rank's seeded instances from bench.make_workload, output tensors shaped like the
    tracker's (x [B,S,N] c128, status [B,S] i32, counters [B,S,4] i32, resid [B,S,2] f64) filled with
    values that encode (instance, track), and the gather bench runs after the timed region."""
    import argparse
    import sys
    import numpy as np
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    args = argparse.Namespace(instances=0, total_instances=total)
    lo, hi = bench.instance_range(args, rank, world)
    d, start, p0, p1s, _, _ = bench.make_workload("p3p", lo, hi)
    B, S, N = p1s.shape[0], start.shape[0], start.shape[1]
    inst = torch.arange(lo, hi, dtype=torch.float64)[:, None, None]
    trk = torch.arange(S, dtype=torch.float64)[None, :, None]
    x = (inst * 1000 + trk + torch.arange(N, dtype=torch.float64)[None, None, :] / 10).to(torch.complex128)
    status = (torch.arange(lo, hi, dtype=torch.int32)[:, None] % 7).repeat(1, S)
    ctr = torch.stack([status, status + 1, status + 2, status + 3], -1)
    resid = inst.repeat(1, S, 2) + trk.repeat(B, 1, 2) / 100
    from paper_2112_03444_b200.distributed import gather_to_rank0
    out = gather_to_rank0([x, status, ctr, resid])
    if rank == 0:
        q.put([o.numpy() for o in out] + [np.asarray(p1s)])
    else:
        q.put([np.asarray(p1s)])
    dist.barrier()
    dist.destroy_process_group()


def test_bench_rank_workloads_and_gather_gloo():
    total, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180), q.get(timeout=180)]
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    full = max(got, key=len)
    other = min(got, key=len)
    x, status, ctr, resid, p1_rank0 = full
    assert x.shape[0] == total and status.shape[0] == total and ctr.shape[0] == total and resid.shape[0] == total
    assert x.dtype.name == "complex128" and status.dtype.name == "int32" and resid.dtype.name == "float64"
    assert (x[:, 0, 0].real == 1000 * torch.arange(total).numpy()).all()
    assert (status[:, 0] == torch.arange(total).numpy() % 7).all() and (ctr[..., 3] == status + 3).all()
    # ranks own disjoint, contiguous blocks of the same seeded instances as one process would build
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import numpy as np
    whole = bench.make_workload("p3p", 0, total)[3]
    assert np.array_equal(np.concatenate([p1_rank0, other[0]]), whole)
