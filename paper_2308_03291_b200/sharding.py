"""Batch data-parallelism across GPUs.

Structures are independent (dist.py:355-361), so a global batch is split
into contiguous per-rank shards with no data-path collective; the only
exchange is an all-gather of the per-structure log Z (and status) so every
rank holds the global vector.  One process per GPU (torch.distributed, NCCL
on B200; gloo works for the same host logic on CPU).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [start, stop) of rank `rank`; the first
    `global_batch % world` ranks take one extra structure."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_shards(local: torch.Tensor, global_batch: int, group=None) -> torch.Tensor:
    """All-gather variable-size 1-D shards (log Z or status) in rank order."""
    world = dist.get_world_size(group)
    sizes = [shard_range(global_batch, world, r) for r in range(world)]
    cap = max(b - a for a, b in sizes)
    buf = torch.zeros(cap, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    out = torch.empty(world * cap, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[r * cap: r * cap + (b - a)] for r, (a, b) in enumerate(sizes)])


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Step time of a multi-GPU run = the slowest rank (timing rule)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
