"""World-size-2 gloo test of the batch-sharding host logic: the
shards cover the global batch, the log-Z all-gather reassembles it in order
(computed here by the CPU oracle per shard), and the step time is the max
over ranks."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_03291_b200.sharding import gather_shards, max_over_ranks, shard_range

HERE = os.path.dirname(os.path.abspath(__file__))


def _worker(rank, world, port, B, q):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    from golden.builders import batch_chain
    from oracle import sd_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(B, world, rank)
    init, tr = batch_chain(100 + a, b - a, 6, 3)  # seeds base + global index
    local = torch.from_numpy(O.chain_log_partition(init, tr))
    full = gather_shards(local, B)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        q.put((full.numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_batch():
    for B in (1, 7, 32, 33):
        for world in (1, 2, 3, 8):
            rs = [shard_range(B, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


def test_gloo_world2_gather_and_max():
    sys.path.insert(0, HERE)
    from golden.builders import batch_chain
    from oracle import sd_oracle as O

    B, world = 7, 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, t = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # reference: every structure seeded by its global index
    ref = np.array([O.chain_log_partition(*batch_chain(100 + i, 1, 6, 3))[0] for i in range(B)])
    np.testing.assert_allclose(full, ref, rtol=1e-12)
    assert t == 2.0
