"""GPU parity: projective spanning trees (Eisner inside/outside,
spanning.py:183-280) and the Kuhlmann argmax (spanning.py:339-402), plus the
spanning-tree flag dispatch through the public API for all 8 flag triples."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_spanning
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("spanning"), ids=lambda c: str(c.meta))
def test_spanning_golden_api(case):
    need_gpu()
    m = case.meta
    d = sd.SpanningTreeCRF(inputs(case)["adjacency"], directed=m["directed"], projective=m["projective"],
                           single_root_edge=m["single"])
    z, algo = sd.log_partition_info(d)
    close_logz(z, case.logz)
    if case.vacuous:
        with pytest.raises(sd.VacuousDistribution):
            sd.marginals(d)
        return
    marg, algo2 = sd.marginals_info(d)
    assert algo2 == algo
    case.check_marg("adjacency", marg["adjacency"], RTOL, ATOL)
    if "argmax_adjacency" in case:  # Kuhlmann (projective) / Chu-Liu-Edmonds (non-projective)
        ind, score, aalgo = sd.argmax_info(d)
        np.testing.assert_array_equal(ind["adjacency"], case["argmax_adjacency"])
        assert score == float(case.argmax_score)
        assert aalgo == case.meta["argmax_algo"]


@pytest.mark.parametrize("single", [False, True])
@pytest.mark.parametrize("B,n", [(4, 128), (6, 9), (3, 1), (3, 2), (2, 50), (2, 160), (1, 203)])  # n > 128: eisner_gen.cu
def test_eisner_batched_vs_oracle(B, n, single):
    need_gpu()
    adj = batch_spanning(3000, B, n)
    logz, marg, st = K.eisner(dev(adj), single)
    assert (st.cpu().numpy() == 0).all()
    heads, score, st2 = K.kuhlmann(dev(adj), single)
    for b in range(B):
        z, mg = O.eisner_marginals(adj[b], single)
        assert abs(logz[b].item() - z) <= RTOL * max(1, abs(z))
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        np.testing.assert_array_equal(heads[b].cpu().numpy(), O.kuhlmann_heads(adj[b], single))


def test_eisner_config_invariants():
    """C4 shape: each dependent has exactly one head (incoming marginals sum
    to 1), multi-root."""
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(0)
    adj = torch.randn(256, 129, 129, device="cuda", generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(129, device="cuda")
    adj[:, i, i] = NEG_INF
    logz, marg, st = K.eisner(adj)
    assert (st == 0).all()
    col = marg.double().sum(1)[:, 1:]
    assert torch.allclose(col, torch.ones_like(col), atol=1e-4)


def test_eisner_zero_ties():
    """Ties on all-zero potentials: Kuhlmann's first-maximum rule."""
    need_gpu()
    adj = np.zeros((1, 6, 6))
    adj[:, :, 0] = NEG_INF
    adj[:, np.arange(6), np.arange(6)] = NEG_INF
    for single in (False, True):
        heads, _, st = K.kuhlmann(dev(adj), single)
        np.testing.assert_array_equal(heads[0].cpu().numpy(), O.kuhlmann_heads(adj[0], single))


@pytest.mark.parametrize("single", [False, True])
def test_cle_argmax_vs_oracle(single):
    """Chu-Liu-Edmonds (spanning.py:410-509), bit-exact arcs at C3 size."""
    need_gpu()
    adj = batch_spanning(3100, 6, 128)
    heads, st = K.cle(dev(adj), single)
    assert (st.cpu().numpy() == 0).all()
    for b in range(6):
        np.testing.assert_array_equal(heads[b].cpu().numpy(), O.cle_heads(adj[b], single))
    # small instances with many cycles (all-equal weights -> ties everywhere)
    z = np.zeros((4, 8, 8))
    z[:, :, 0] = -np.inf
    for b in range(4):
        np.fill_diagonal(z[b], -np.inf)
    z[1] = batch_spanning(5, 1, 7)[0]
    heads, st = K.cle(dev(z), single)
    for b in range(4):
        np.testing.assert_array_equal(heads[b].cpu().numpy(), O.cle_heads(z[b], single))


@pytest.mark.parametrize("single", [False, True])
def test_eisner_exp_space_fallback(single):
    """Instances whose linear-space charts over/underflow (huge |theta|) are
    recomputed by the log-space kernel; mixed batch with normal instances."""
    need_gpu()
    adj = batch_spanning(3200, 4, 40)
    adj[1] *= 80.0   # ~e^{+-250} per arc: linear space must give up
    adj[3][adj[3] > 0] *= 50.0
    logz, marg, st = K.eisner(dev(adj), single)
    assert (st.cpu().numpy() == 0).all()
    for b in range(4):
        z, mg = O.eisner_marginals(adj[b], single)
        assert abs(logz[b].item() - z) <= RTOL * abs(z) + 1e-6
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


def test_eisner_kuhlmann_concurrent():
    """Fused request (Eisner on the current stream, Kuhlmann on a side
    stream) == the two separate calls."""
    need_gpu()
    adj = dev(batch_spanning(3100, 6, 40))
    (lz, mg, st), (heads, score, st2) = K.eisner_kuhlmann(adj)
    lz1, mg1, _ = K.eisner(adj)
    heads1, score1, _ = K.kuhlmann(adj)
    torch.cuda.synchronize()
    assert torch.equal(lz, lz1) and torch.equal(mg, mg1)
    assert torch.equal(heads, heads1) and torch.equal(score, score1)
