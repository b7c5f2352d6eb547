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
