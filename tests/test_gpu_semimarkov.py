"""GPU parity: semi-Markov CRF (chain.py:250-327) through the C-ABI."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_semi_markov
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("semi_markov"), ids=lambda c: str(c.meta))
def test_semimarkov_golden(case):
    need_gpu()
    d = sd.SemiMarkovCRF(inputs(case)["segment_potentials"])
    close_logz(sd.log_partition(d), case.logz)
    marg, algo = sd.marginals_info(d)
    assert algo == "semi-markov-forward"
    case.check_marg("segment_potentials", marg["segment_potentials"], RTOL, ATOL)
    ind, score, algo = sd.argmax_info(d)
    assert algo == "semi-markov-viterbi"
    np.testing.assert_array_equal(ind["segment_potentials"], case["argmax_segment_potentials"])
    assert score == float(case.argmax_score)


@pytest.mark.parametrize("B,n,s,m", [(3, 64, 8, 32), (4, 10, 3, 5), (2, 1, 1, 3), (2, 20, 20, 2)])
def test_semimarkov_batched_vs_oracle(B, n, s, m):
    need_gpu()
    th = batch_semi_markov(7000, B, n, s, m)
    logz, marg, st = K.semimarkov_fb(dev(th))
    seg, cnt, score, st2 = K.semimarkov_viterbi(dev(th))
    for b in range(B):
        z, mg = O.sm_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        segs, sc = O.sm_viterbi(th[b])
        got = [tuple(int(v) for v in r) for r in seg[b].cpu().numpy()[: cnt[b].item()]]
        assert got == [tuple(x) for x in segs]  # bit-exact
        assert score[b].item() == sc


def test_semimarkov_coverage_invariant():
    """Each position is covered by exactly one segment (test_chain.py:133-142)."""
    need_gpu()
    th = batch_semi_markov(1, 4, 64, 8, 32)
    logz, marg, st = K.semimarkov_fb(dev(th))
    mg = marg.double().sum((3, 4))  # [B, n, s]
    n, s = 64, 8
    cover = torch.zeros(4, n, dtype=torch.float64, device="cuda")
    for t in range(n):
        for w in range(1, s + 1):
            if t + w <= n:
                cover[:, t:t + w] += mg[:, t, w - 1, None]
    assert torch.allclose(cover, torch.ones_like(cover), atol=1e-4)
