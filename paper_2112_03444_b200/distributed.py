"""Multi-GPU sharding of tracks x instances.

Instances are independent ("HC follows many independent tracks"): rank g of G owns
the contiguous instance block [g*B/G, (g+1)*B/G) with all S tracks each; start solutions
and p0 are replicated.  Tracking needs no communication; the only collective is the final
gather of solutions/statuses/counters/residuals to rank 0 (NCCL on GPUs, gloo in CPU tests).
"""
from __future__ import annotations

import os


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced block [lo, hi) of n_total items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def sharded_settings(st):
    """Tracker settings for a job sharded over GPUs: the lane layout pinned to the throughput layout
    when left on HC_LAYOUT_AUTO (whose choice depends on the batch size for N <= 16), so every track
    gives the same bits for any shard size or GPU count (include/hc.h, Determinism)."""
    from . import hc
    if st.lane_layout == hc.HC_LAYOUT_AUTO:
        st.lane_layout = hc.HC_LAYOUT_THROUGHPUT
    return st


def env_rank_world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (1 process when unset)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def gather_to_rank0(tensors, group=None):
    """Gather each tensor of `tensors` (same shapes on every rank along dim 0 except possibly the
    first dimension) to rank 0.  Returns the list of concatenated tensors on rank 0, None elsewhere.

    Uneven first dimensions are padded to the max and trimmed after the gather, so one
    `torch.distributed.gather` per tensor suffices (NCCL: send/recv based gather)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out = []
    for t in tensors:
        t = t.contiguous()
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes)
        if t.shape[0] < m:
            pad = torch.zeros((m - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            t = torch.cat([t, pad])
        # complex tensors travel as their real view (NCCL has no complex dtype)
        send = torch.view_as_real(t) if t.is_complex() else t
        bufs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
        dist.gather(send, bufs, dst=0, group=group)
        if rank == 0:
            parts = [torch.view_as_complex(b) if t.is_complex() else b for b in bufs]
            out.append(torch.cat([p[: sizes[i]] for i, p in enumerate(parts)]))
    return out if rank == 0 else None
