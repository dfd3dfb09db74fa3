"""GPU parity: linear-chain CRF (chain.py:64-114) through the C-ABI."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_chain
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("chain"), ids=lambda c: str(c.meta))
def test_chain_golden(case):
    need_gpu()
    x = inputs(case)
    d = sd.LinearChainCRF(x["init"], x["transitions"])
    close_logz(sd.log_partition(d), case.logz)
    if case.vacuous:
        with pytest.raises(sd.VacuousDistribution):
            sd.marginals(d)
        with pytest.raises(sd.VacuousDistribution):
            sd.argmax(d)
        return
    marg, algo = sd.marginals_info(d)
    assert algo == "forward"
    case.check_marg("init", marg["init"], RTOL, ATOL)
    case.check_marg("transitions", marg["transitions"], RTOL, ATOL)
    ind, score, algo = sd.argmax_info(d)
    assert algo == "viterbi"
    np.testing.assert_array_equal(ind["init"], case["argmax_init"])
    np.testing.assert_array_equal(ind["transitions"], case["argmax_transitions"])
    assert score == float(case.argmax_score)


@pytest.mark.parametrize("B,n,m", [(32, 128, 32), (5, 40, 7), (3, 2, 64), (4, 1, 3), (2, 300, 130)])
def test_chain_batched_vs_oracle(B, n, m):
    need_gpu()
    init, tr = batch_chain(100, B, n, m)
    logz, mi, mt, st = K.chain_fb(dev(init), dev(tr))
    z, pi, pt = O.chain_marginals(init, tr)
    assert (st.cpu().numpy() == 0).all()
    np.testing.assert_allclose(logz.cpu().numpy(), z, rtol=RTOL)
    np.testing.assert_allclose(mi.cpu().numpy(), pi, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(mt.cpu().numpy(), pt, rtol=RTOL, atol=ATOL)
    tags, score, st2 = K.chain_viterbi(dev(init), dev(tr))
    otags, oscore = O.chain_viterbi(init, tr)
    np.testing.assert_array_equal(tags.cpu().numpy(), otags)  # bit-exact argmax
    np.testing.assert_array_equal(score.cpu().numpy(), oscore)


def test_chain_config_invariants():
    """C1 shape: per-step marginals sum to 1, tag marginals sum to 1
    (test_chain.py:46-56)."""
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(0)
    init = torch.randn(32, 32, device="cuda", generator=g)
    tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
    logz, mi, mt, st = K.chain_fb(init, tr)
    assert (st == 0).all()
    s = mt.double().sum(dim=(2, 3))
    assert torch.allclose(s, torch.ones_like(s), atol=1e-4)
    assert torch.allclose(mi.double().sum(1), torch.ones(32, dtype=torch.float64, device="cuda"), atol=1e-4)


def test_chain_status_codes():
    need_gpu()
    init = np.zeros((3, 2))
    tr = np.zeros((3, 2, 2, 2))
    tr[1] = NEG_INF  # vacuous
    tr[2, 0, 0, 0] = np.nan  # invalid
    logz, _, _, st = K.chain_fb(dev(init), dev(tr))
    assert st.cpu().tolist() == [0, 1, 2]
    assert logz[1].item() == NEG_INF
    _, _, st2 = K.chain_viterbi(dev(init), dev(tr))
    assert st2.cpu().tolist() == [0, 1, 2]


def test_chain_padding_neutral():
    """chain.py:161-176 identity padding leaves log Z unchanged."""
    need_gpu()
    init, tr = batch_chain(7, 1, 6, 3)
    pad = np.full((1, 4, 3, 3), NEG_INF)
    for i in range(3):
        pad[:, :, i, i] = 0.0
    z0 = K.chain_fb(dev(init), dev(tr), False)[0].item()
    z1 = K.chain_fb(dev(init), dev(np.concatenate([tr, pad], 1)), False)[0].item()
    assert abs(z0 - z1) < 1e-5


def test_batch_map_matches_singles():
    need_gpu()
    ds = [sd.LinearChainCRF(*[x[0] for x in batch_chain(s, 1, 5, 3)]) for s in range(4)]
    zs = sd.batch_map(sd.log_partition, ds)
    for d, z in zip(ds, zs):
        assert abs(z - sd.log_partition(d)) < 1e-9


def test_chain_fb_viterbi_concurrent():
    """The fused request (forward-backward on the current stream, Viterbi on a
    side stream) returns exactly what the two separate calls return."""
    need_gpu()
    init, tr = batch_chain(300, 32, 128, 32)
    (lz, mi, mt, st), (tags, score, st2) = K.chain_fb_viterbi(dev(init), dev(tr))
    lz1, mi1, mt1, _ = K.chain_fb(dev(init), dev(tr))
    tags1, score1, _ = K.chain_viterbi(dev(init), dev(tr))
    torch.cuda.synchronize()
    assert torch.equal(lz, lz1) and torch.equal(mt, mt1) and torch.equal(mi, mi1)
    assert torch.equal(tags, tags1) and torch.equal(score, score1)
    assert (st == 0).all() and (st2 == 0).all()


def test_chain_linear_fallback_mixed_batch():
    """C1-shaped batch (linear recurrence path) where some instances cannot be
    held in scaled linear fp32: huge potentials, and -inf structure late in
    the chain (zero states in the BACKWARD pass only).  They are recomputed
    by the exact log-space path; every instance must match the oracle."""
    need_gpu()
    init, tr = batch_chain(310, 4, 128, 32)
    tr[1] *= 30.0                       # exp(theta) over/underflows fp32: beyond the linear range
    tr[2, 120, :, 1:] = NEG_INF         # step 120: only tag 0 reachable -> zeros in beta
    tr[3, 5, :, :] -= 200.0             # one very unlikely step (uniform shift)
    logz, mi, mt, st = K.chain_fb(dev(init), dev(tr))
    assert (st.cpu().numpy() == 0).all()
    for b in range(4):
        z, pi, pt = O.chain_marginals(init[b:b + 1], tr[b:b + 1])
        assert abs(logz[b].item() - z[0]) <= RTOL * abs(z[0])
        np.testing.assert_allclose(mi[b].cpu().numpy(), pi[0], rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(mt[b].cpu().numpy(), pt[0], rtol=RTOL, atol=ATOL)
