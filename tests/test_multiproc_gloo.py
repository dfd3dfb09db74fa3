"""World-size-2 gloo test of the batch-sharding host logic: the
shards cover the global batch, the log-Z all-gather reassembles it in order
(computed here by the CPU oracle per shard), and the step time is the max
over ranks."""

import os
import sys

import numpy as np
import pytest
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


def _gpu_worker(rank, world, port, q):
    """Both ranks on cuda:0 (independent kernels, nothing waits across ranks):
    the product sharding entry runs the real sm_100a kernels on each shard and
    all-gathers log Z / status over gloo."""
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import paper_2308_03291_b200 as sd
    from golden.builders import alignment, batch_alignment
    from paper_2308_03291_b200 import kernels as K

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    B = 7
    th = torch.from_numpy(batch_alignment(600, B, 20, 9)).float().pin_memory()
    res = sd.run_sharded(K.nw_fb, [th])
    torch.cuda.synchronize()
    dists = [sd.MonotoneAlignmentCRF(alignment(700 + i, 6 + i, 5)) for i in range(5)]
    lz = sd.sharded_batch_map(sd.log_partition, dists)
    mg = sd.sharded_batch_map(sd.marginals, dists, gather=False)
    if rank == 0:
        q.put((res.logz.cpu().numpy(), res.status.cpu().numpy(), (res.start, res.stop),
               res.local[1].cpu().numpy(), lz, [m is not None for m in mg]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_real_kernels():
    import paper_2308_03291_b200 as sd
    from golden.builders import alignment, batch_alignment
    from paper_2308_03291_b200 import kernels as K

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 31000 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    logz, status, (a, b), marg0, lz, owned = q.get()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    th = torch.from_numpy(batch_alignment(600, 7, 20, 9)).float().cuda()
    z1, m1, st1 = K.nw_fb(th)
    np.testing.assert_array_equal(logz, z1.cpu().numpy())  # same kernels, same shards -> identical
    np.testing.assert_array_equal(status, st1.cpu().numpy())
    assert (a, b) == (0, 4)
    np.testing.assert_array_equal(marg0, m1[a:b].cpu().numpy())
    dists = [sd.MonotoneAlignmentCRF(alignment(700 + i, 6 + i, 5)) for i in range(5)]
    assert lz == [sd.log_partition(d) for d in dists]
    assert owned == [True, True, True, False, False]
