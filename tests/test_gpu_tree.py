"""GPU parity: Tree-CRF CKY (constituency.py:52-133) through the C-ABI."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_tree
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("tree"), ids=lambda c: str(c.meta))
def test_tree_golden(case):
    need_gpu()
    d = sd.TreeCRF(inputs(case)["span_potentials"])
    close_logz(sd.log_partition(d), case.logz)
    marg, algo = sd.marginals_info(d)
    assert algo == "cky-inside"
    case.check_marg("span_potentials", marg["span_potentials"], RTOL, ATOL)
    ind, score, algo = sd.argmax_info(d)
    assert algo == "max-plus-cky"
    np.testing.assert_array_equal(ind["span_potentials"], case["argmax_span_potentials"])
    assert score == float(case.argmax_score)


@pytest.mark.parametrize("B,n,m", [(3, 64, 32), (4, 17, 5), (2, 1, 3), (2, 128, 4), (3, 33, 33), (2, 20, 16), (2, 12, 64),
                                   (2, 80, 8), (2, 160, 6), (1, 257, 3)])  # n > 128: tree_gen.cu
def test_tree_batched_vs_oracle(B, n, m):
    need_gpu()
    th = batch_tree(4000, B, n, m)
    logz, marg, st = K.tree_fb(dev(th))
    assert (st.cpu().numpy() == 0).all()
    lz0, _, _ = K.tree_fb(dev(th), marginals=False)
    labels, score, _ = K.tree_viterbi(dev(th))
    for b in range(B):
        z, mg = O.tree_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        assert abs(lz0[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        lab, sc = O.tree_argmax(th[b])
        np.testing.assert_array_equal(labels[b].cpu().numpy(), lab)  # bit-exact
        assert score[b].item() == sc


def test_tree_general_status():
    """n > 128 (tree_gen.cu): invalid, vacuous and masked instances."""
    need_gpu()
    n, m = 140, 4
    th = batch_tree(4100, 4, n, m)
    th[0, 5, 90, 2] = np.nan            # invalid
    th[1, 0, n - 1, :] = NEG_INF        # the root span has no label -> vacuous
    th[2, :, :, 1:] = NEG_INF           # one label everywhere
    th[2, 10, 50, 0] = NEG_INF          # and one span forbidden
    logz, marg, st = K.tree_fb(dev(th))
    labels, score, st2 = K.tree_viterbi(dev(th))
    assert st.cpu().tolist() == [2, 1, 0, 0] and st2.cpu().tolist() == [2, 1, 0, 0]
    assert float(marg[1].abs().sum()) == 0.0 and (labels[1] == -1).all()
    for b in (2, 3):
        z, mg = O.tree_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        lab, sc = O.tree_argmax(th[b])
        np.testing.assert_array_equal(labels[b].cpu().numpy(), lab)
        assert score[b].item() == sc


def test_tree_config_invariants():
    """C5a shape: Tree-CRF marginals sum to 2n-1 nodes (test_constituency.py:39-42)."""
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(0)
    th = torch.randn(128, 64, 64, 32, device="cuda", generator=g)
    logz, marg, st = K.tree_fb(th)
    assert (st == 0).all()
    tot = marg.double().sum((1, 2, 3))
    assert torch.allclose(tot, torch.full_like(tot, 127.0), rtol=1e-4)
    assert float(torch.tril(marg.sum(-1), -1).abs().sum()) == 0.0


def test_tree_status():
    need_gpu()
    th = batch_tree(1, 3, 4, 2)
    th[1, 0, 3, :] = NEG_INF  # root span forbidden -> vacuous
    th[2, 1, 2, 0] = np.inf
    logz, marg, st = K.tree_fb(dev(th))
    assert st.cpu().tolist() == [0, 1, 2]


def test_tree_linear_fallback_mixed_batch():
    """Instances the scaled-linear charts cannot hold (huge / very uneven
    potentials, -inf spans) are redone in log space; the rest of the batch
    stays on the linear path.  Every instance must match the oracle."""
    need_gpu()
    th = batch_tree(4100, 5, 24, 8)
    th[1] *= 300.0               # folds spread over hundreds of nats -> linear range exceeded
    th[3, 2, 9, :] = NEG_INF     # one forbidden span: exact -inf structure
    th[4, :, :, 0] += 60.0       # uniform shift: still linear-representable
    logz, marg, st = K.tree_fb(dev(th))
    lz0, _, st0 = K.tree_fb(dev(th), marginals=False)
    assert (st.cpu().numpy() == 0).all() and (st0.cpu().numpy() == 0).all()
    for b in range(th.shape[0]):
        z, mg = O.tree_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        assert abs(lz0[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
