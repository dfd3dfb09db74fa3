"""GPU parity: CTC (alignment.py:231-336) through the C-ABI."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_ctc
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("ctc"), ids=lambda c: str(c.meta))
def test_ctc_golden(case):
    need_gpu()
    x = inputs(case)
    d = sd.CTCDist(x["frame_potentials"], tuple(int(t) for t in x["target"]))
    close_logz(sd.log_partition(d), case.logz)
    if case.vacuous:
        with pytest.raises(sd.VacuousDistribution):
            sd.marginals(d)
        return
    marg, algo = sd.marginals_info(d)
    assert algo == "ctc-forward"
    case.check_marg("frame_potentials", marg["frame_potentials"], RTOL, ATOL)
    ind, score, algo = sd.argmax_info(d)
    assert algo == "max-plus-ctc"
    np.testing.assert_array_equal(ind["frame_potentials"], case["argmax_frame_potentials"])
    assert score == float(case.argmax_score)


# the last three run ctc_gen.cu: 2L+1 > 1024 states, a 20000-word vocabulary
@pytest.mark.parametrize("B,T,V,L", [(4, 512, 128, 128), (3, 50, 7, 12), (2, 9, 3, 4), (5, 1, 4, 0), (2, 30, 40, 300),
                                     (2, 1100, 30, 520), (2, 700, 6, 600), (2, 40, 20000, 10)])
def test_ctc_batched_vs_oracle(B, T, V, L):
    need_gpu()
    fp, tg = batch_ctc(1000, B, T, V, L)
    logz, marg, st = K.ctc_fb(dev(fp), dev(tg, torch.int32))
    z, mg = O.ctc_marginals(fp, tg)
    vac = np.isneginf(z)
    np.testing.assert_array_equal(st.cpu().numpy(), vac.astype(np.int32))
    lz = logz.cpu().numpy()
    assert np.all(lz[vac] == NEG_INF)
    np.testing.assert_allclose(lz[~vac], z[~vac], rtol=RTOL)
    np.testing.assert_allclose(marg.cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
    lz2, _, _ = K.ctc_fb(dev(fp), dev(tg, torch.int32), marginals=False)
    np.testing.assert_allclose(lz2.cpu().numpy()[~vac], z[~vac], rtol=RTOL)
    labs, score, st2 = K.ctc_viterbi(dev(fp), dev(tg, torch.int32))
    olabs, oscore = O.ctc_argmax(fp, tg)
    ok = ~vac
    np.testing.assert_array_equal(labs.cpu().numpy()[ok], olabs[ok])  # bit-exact
    np.testing.assert_array_equal(score.cpu().numpy()[ok], oscore[ok])


def test_ctc_frame_sums_config():
    """C2b shape: per-frame marginals sum to 1 (test_alignment.py:99-102)."""
    need_gpu()
    B, T, V, L = 256, 512, 128, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    fp = torch.randn(B, T, V, device="cuda", generator=g)
    tg = torch.randint(1, V, (B, L), device="cuda", generator=g, dtype=torch.int32)
    logz, marg, st = K.ctc_fb(fp, tg)
    ok = st == 0
    s = marg.double().sum(-1)[ok]
    assert torch.allclose(s, torch.ones_like(s), atol=1e-4)


def test_ctc_status():
    need_gpu()
    fp = np.zeros((3, 2, 3))
    tg = np.array([[1, 2], [1, 1], [1, 2]])  # [1,1] infeasible in 2 frames
    fp[2, 0, 1] = np.nan
    logz, _, st = K.ctc_fb(dev(fp), dev(tg, torch.int32))
    assert st.cpu().tolist() == [0, 1, 2]


@pytest.mark.parametrize("scale,exact", [(25.0, False), (400.0, True)])
def test_ctc_large_magnitudes(scale, exact):
    """Emission log-potentials scaled to |theta| ~ 25 nats per frame (|log Z| ~ 1e4): the
    fp32 (value, integer offset) recursion keeps the parity bar, every stored value being
    renormalised to |v| <= 1/2 around an exact integer offset.  Its per-step rounding grows
    like |theta| 2^-24, so at |theta| ~ 400 nats over 300 frames (|log Z| ~ 2e5) fp32
    drifts past 1e-4 and float64 potentials take the exact kernels instead."""
    need_gpu()
    fp, tg = batch_ctc(2000, 3, 300, 40, 60)
    fp = (fp * scale).astype(np.float32).astype(np.float64)  # the oracle sees the kernel's inputs
    x = torch.as_tensor(fp, dtype=torch.float64 if exact else torch.float32, device="cuda")
    logz, marg, st = K.ctc_fb(x, dev(tg, torch.int32))
    z, mg = O.ctc_marginals(fp, tg)
    ok = ~np.isneginf(z)
    assert ok.any()
    np.testing.assert_allclose(logz.cpu().numpy()[ok], z[ok], rtol=RTOL)
    np.testing.assert_allclose(marg.cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
