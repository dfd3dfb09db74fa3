"""Batch data-parallelism across GPUs: the sharded counterpart
of the reference's serial `batch_map` (dist.py:355-361).

Structures are independent, so a global batch is split into contiguous
per-rank shards with no data-path collective; the only exchange is an
all-gather of the per-structure log Z and status so every rank holds the
global vectors (marginals stay on the GPU that computed them).  One process
per GPU under torch.distributed (NCCL on B200; the same host logic runs on
gloo, where the gathered tensors travel through host memory).

    import torch.distributed as dist
    from paper_2308_03291_b200 import kernels as K, sharding
    res = sharding.run_sharded(K.nw_fb, [theta_host])   # every rank: res.logz = log Z of the global batch
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def _world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [start, stop) of rank `rank`; the first
    `global_batch % world` ranks take one extra structure."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_shards(local: torch.Tensor, global_batch: int, group=None) -> torch.Tensor:
    """All-gather variable-size 1-D shards (log Z or status) in rank order.
    NCCL gathers device tensors in place; other backends (gloo) gather host
    copies and the result is moved back to `local`'s device."""
    world = dist.get_world_size(group)
    sizes = [shard_range(global_batch, world, r) for r in range(world)]
    cap = max(b - a for a, b in sizes)
    on_host = dist.get_backend(group) != "nccl"
    src = local.cpu() if on_host else local
    buf = torch.zeros(cap, dtype=src.dtype, device=src.device)
    buf[: src.numel()] = src
    out = torch.empty(world * cap, dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    full = torch.cat([out[r * cap: r * cap + (b - a)] for r, (a, b) in enumerate(sizes)])
    return full.to(local.device) if on_host else full


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Step time of a multi-GPU run = the slowest rank (timing rule)."""
    on_host = dist.get_backend(group) != "nccl"
    t = torch.tensor([float(value)], dtype=torch.float64, device=None if on_host else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


@dataclass
class ShardResult:
    start: int            # this rank's shard is [start, stop) of the global batch
    stop: int
    logz: torch.Tensor    # [global_batch] float64, every rank
    status: torch.Tensor  # [global_batch] int32, every rank
    local: tuple          # the kernel's outputs for the local shard (marginals stay on this GPU)


def run_sharded(fn, inputs, *, group=None, local_inputs: bool = False, global_batch: int | None = None):
    """Run a batched kernel entry (`kernels.*_fb`, `kernels.mtt`, ...; it
    returns (logz, ..., status)) over this rank's shard of a global batch.

    `inputs` are tensors whose leading axis is the GLOBAL batch (host --
    ideally pinned -- or device); each rank copies only its slice to its
    current CUDA device.  With `local_inputs=True` they are already this
    rank's shard (then `global_batch` must be given).  Returns a
    ShardResult whose log Z / status cover the global batch on every rank."""
    world, rank = _world(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    if local_inputs:
        if global_batch is None:
            raise ValueError("global_batch is required with local_inputs")
        B = int(global_batch)
        a, b = shard_range(B, world, rank)
        if inputs[0].shape[0] != b - a:
            raise ValueError(f"rank {rank}: local shard has {inputs[0].shape[0]} structures, expected {b - a}")
        xs = [t.to(dev, non_blocking=True) for t in inputs]
    else:
        B = int(inputs[0].shape[0])
        a, b = shard_range(B, world, rank)
        xs = [t[a:b].to(dev, non_blocking=True) for t in inputs]
    out = fn(*xs)
    logz, status = out[0], out[-1]
    if world > 1:
        logz = gather_shards(logz, B, group)
        status = gather_shards(status, B, group)
    return ShardResult(a, b, logz, status, tuple(out))


def sharded_batch_map(op, dists, *args, group=None, gather: bool = True, **kwargs) -> list:
    """`dist.batch_map` over the ranks: rank r maps `op` over its contiguous
    shard of `dists` (one grouped GPU launch per shape group, dist.py:355-361
    semantics) and, with `gather`, every rank receives the full result list
    in the original order (all_gather_object); without it the other ranks'
    entries are None."""
    from .dist import batch_map

    dists = list(dists)
    world, rank = _world(group)
    a, b = shard_range(len(dists), world, rank)
    local = batch_map(op, dists[a:b], *args, **kwargs)
    if world == 1:
        return local
    if not gather:
        return [None] * a + local + [None] * (len(dists) - b)
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return [r for p in parts for r in p]
