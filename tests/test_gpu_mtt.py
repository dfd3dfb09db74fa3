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
    case.check_marg("adjacency", marg[0].cpu().numpy(), RTOL, 2e-6)


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
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=1e-5 if single else 2e-6)


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
