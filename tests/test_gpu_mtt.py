"""GPU parity: Matrix-Tree non-projective spanning trees (spanning.py:90-175)."""

import numpy as np
import pytest
import torch

from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_spanning, spanning
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu

CASES = [c for c in load("spanning") if not c.meta["projective"]]


@pytest.mark.parametrize("case", CASES, ids=lambda c: str(c.meta))
def test_mtt_golden_kernel(case):
    need_gpu()
    adj = inputs(case)["adjacency"]
    single = case.meta["single"]
    logz, marg, st = K.mtt(dev(adj[None]), single)
    close_logz(logz[0].item(), case.logz)
    if case.vacuous:
        assert st[0].item() == 1
        return
    assert st[0].item() == 0
    case.check_marg("adjacency", marg[0].cpu().numpy(), RTOL, ATOL)


@pytest.mark.parametrize("single", [False, True])
@pytest.mark.parametrize("B,n", [(8, 128), (5, 37), (3, 1), (4, 2), (3, 100)])
def test_mtt_batched_vs_oracle(B, n, single):
    need_gpu()
    adj = batch_spanning(2000, B, n)
    logz, marg, st = K.mtt(dev(adj), single)
    assert (st.cpu().numpy() == 0).all()
    for b in range(B):
        z = O.mtt_log_partition(adj[b], single)
        assert abs(logz[b].item() - z) <= RTOL * max(1, abs(z))
        mg = O.mtt_marginals(adj[b], single)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


def test_mtt_config_invariants():
    """C3 shape: every dependent's incoming marginals sum to 1; column
    shift invariance of log Z (test_spanning.py:78-86)."""
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(0)
    adj = torch.randn(512, 129, 129, device="cuda", generator=g)
    adj[:, :, 0] = NEG_INF
    idx = torch.arange(129, device="cuda")
    adj[:, idx, idx] = NEG_INF
    logz, marg, st = K.mtt(adj)
    assert (st == 0).all()
    col = marg.double().sum(1)[:, 1:]
    assert torch.allclose(col, torch.ones_like(col), atol=1e-4)
    adj2 = adj.clone()
    adj2[:, :, 1:] += 3.7
    z2, _, _ = K.mtt(adj2, marginals=False)
    assert torch.allclose(z2 - 128 * 3.7, logz, rtol=1e-5)


def test_mtt_status():
    need_gpu()
    adj = batch_spanning(3, 3, 5)
    adj[1, :, 2] = NEG_INF  # node 2 has no incoming edge
    adj[2, 1, 3] = np.nan
    logz, marg, st = K.mtt(dev(adj))
    assert st.cpu().tolist() == [0, 1, 2]
    assert logz[1].item() == NEG_INF


@pytest.mark.parametrize("single", [False, True])
def test_mtt_cut_off_groups_are_vacuous(single):
    """A group of nodes with finite arcs among themselves but none from the
    rest of the tree makes the Laplacian exactly singular: the reference's
    fp64 pivot test reports -inf (numerics.py:143-146); the kernel's
    structural check must too, whatever fp rounding does."""
    need_gpu()
    rng = np.random.default_rng(77)
    B, n = 64, 20
    adj = batch_spanning(5000, B, n)
    for b in range(B):
        k = int(rng.integers(2, 6))
        grp = 1 + rng.choice(n, size=k, replace=False)
        rest = np.setdiff1d(np.arange(n + 1), grp)
        adj[b][np.ix_(rest, grp)] = NEG_INF  # nothing outside reaches the group
    logz, marg, st = K.mtt(dev(adj), single)
    assert (st.cpu().numpy() == 1).all()
    assert (logz.cpu().numpy() == NEG_INF).all()
    assert (marg.cpu().numpy() == 0).all()
    z2, _, st2 = K.mtt(dev(adj), single, marginals=False)
    assert (st2.cpu().numpy() == 1).all()
    for b in range(4):
        assert O.mtt_log_partition(adj[b], single) == NEG_INF


def test_mtt_single_root_branches():
    """Feasible with several root edges, infeasible with exactly one."""
    need_gpu()
    adj = np.full((2, 5, 5), NEG_INF)
    adj[:, 0, 1] = 0.1
    adj[:, 0, 2] = -0.4
    adj[:, 1, 3] = 0.7
    adj[:, 2, 4] = 0.2
    adj[1, 3, 2] = 0.4  # instance 1: 1 -> 3 -> 2 -> 4 connects the branches
    for single in (False, True):
        logz, marg, st = K.mtt(dev(adj), single)
        for b in range(2):
            z = O.mtt_log_partition(adj[b], single)
            close_logz(logz[b].item(), z)
            assert st[b].item() == (1 if z == NEG_INF else 0)
            if z != NEG_INF:
                np.testing.assert_allclose(marg[b].cpu().numpy(), O.mtt_marginals(adj[b], single), rtol=RTOL,
                                           atol=ATOL)
    assert O.mtt_log_partition(adj[0], True) == NEG_INF


@pytest.mark.parametrize("single", [False, True])
@pytest.mark.parametrize("B,n", [(2, 129), (2, 160), (1, 200)])
def test_mtt_general_n_vs_oracle(B, n, single):
    """n > 128 (beyond the register-resident kernel): the general fp64
    Gauss-Jordan (mtt_gen.cu) through the same entry, vs the oracle."""
    need_gpu()
    adj = batch_spanning(2100, B, n)
    logz, marg, st = K.mtt(dev(adj), single)
    assert (st.cpu().numpy() == 0).all()
    for b in range(B):
        z = O.mtt_log_partition(adj[b], single)
        assert abs(logz[b].item() - z) <= RTOL * max(1, abs(z))
        np.testing.assert_allclose(marg[b].cpu().numpy(), O.mtt_marginals(adj[b], single), rtol=RTOL, atol=ATOL)
    cut = adj.copy()
    cut[:, :, 5] = NEG_INF
    cut[:, 7, 5] = 0.0  # node 5 reachable only from node 7 ...
    cut[:, 5, 7] = 0.0
    cut[:, :, 7] = NEG_INF
    cut[:, 5, 7] = 0.0  # ... which is reachable only from 5: a cut-off 2-cycle
    z2, _, st2 = K.mtt(dev(cut), single)
    assert (st2.cpu().numpy() == 1).all() and (z2.cpu().numpy() == NEG_INF).all()
