"""Instance sharding across ranks and the one collective of the path.

A batch of independent DCOPF instances (config 4) is split into contiguous
shards, one per rank (one process per GPU); the ranks never communicate while
iterating.  After the timed region, the per-instance results (bound, best,
status, ...) are gathered once -- NCCL over NVLink on the GPU box, gloo in the
CPU tests.  Nothing here touches the dual arithmetic.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard(B: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of B instances for `rank` of `world`
    (sizes differ by at most one; earlier ranks take the remainder)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(int(B), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_sizes(B: int, world: int) -> List[int]:
    return [hi - lo for lo, hi in (shard(B, r, world) for r in range(world))]


def gather_instance_results(rows: Sequence, B_total: int, group=None, sizes=None):
    """All-gather per-instance result vectors.

    rows: list of equally-long 1-D tensors (this rank's shard, any dtype
    castable to float64, on the device the process group uses).  Returns a
    float64 tensor [len(rows), B_total] in global instance order, on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = list(sizes) if sizes is not None else shard_sizes(B_total, world)
    assert sum(sizes) == B_total and len(sizes) == world
    n_local = sizes[rank]
    stacked = torch.stack([r.to(torch.float64) for r in rows])
    assert stacked.shape[1] == n_local, (stacked.shape, n_local)
    m = max(sizes)
    pad = torch.full((stacked.shape[0], m), float("nan"), dtype=torch.float64, device=stacked.device)
    pad[:, :n_local] = stacked
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, :sz] for p, sz in zip(parts, sizes)], dim=1)
