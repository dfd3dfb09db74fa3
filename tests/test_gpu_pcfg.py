"""GPU parity: PCFG inside, span marginals, full gradients (rule / root /
emission expected counts) and max-plus argmax (constituency.py:246-371)."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import batch_pcfg
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("pcfg"), ids=lambda c: str(c.meta))
def test_pcfg_golden(case):
    need_gpu()
    x = inputs(case)
    d = sd.PCFG(x["root"], x["binary_rules"], x["emissions"])
    close_logz(sd.log_partition(d), case.logz)
    if case.vacuous:
        with pytest.raises(sd.VacuousDistribution):
            sd.marginals(d)
        return
    marg, algo = sd.marginals_info(d)
    assert algo == "pcfg-inside"
    assert list(marg) == ["sticky"]
    case.check_marg("sticky", marg["sticky"], RTOL, ATOL)


@pytest.mark.parametrize("B,n,nt,pt", [(2, 64, 32, 32), (3, 12, 5, 7), (2, 2, 3, 2), (2, 30, 32, 17)])
def test_pcfg_batched_vs_oracle(B, n, nt, pt):
    need_gpu()
    root, rules, emis = batch_pcfg(4000, B, n, nt, pt)
    logz, marg, st = K.pcfg_fb(dev(root), dev(rules), dev(emis))
    assert (st.cpu().numpy() == 0).all()
    for b in range(min(B, 1 if n > 40 else B)):
        if n > 40:  # oracle outside is slow at n=64: check log Z and the root/leaf identities
            z = O.pcfg_log_partition(root[b], rules[b], emis[b])
            assert abs(logz[b].item() - z) <= RTOL * abs(z)
            continue
        z, g = O.pcfg_gradients(root[b], rules[b], emis[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), g["sticky"], rtol=RTOL, atol=ATOL)


def test_pcfg_config_invariants():
    """C5b shape: root span marginal = 1, each leaf marginal = 1, and the
    span marginals sum to 2n-1 (every binary tree has 2n-1 constituents)."""
    need_gpu()
    root, rules, emis = batch_pcfg(5000, 128, 64, 32, 32)
    logz, marg, st = K.pcfg_fb(dev(root), dev(rules), dev(emis))
    assert (st == 0).all()
    m = marg.double()
    assert torch.allclose(m[:, 0, 63], torch.ones(128, dtype=torch.float64, device="cuda"), atol=1e-4)
    d = torch.diagonal(m, dim1=1, dim2=2)
    assert torch.allclose(d, torch.ones_like(d), atol=1e-4)
    assert torch.allclose(m.sum((1, 2)), torch.full((128,), 127.0, dtype=torch.float64, device="cuda"), rtol=1e-4)


def test_pcfg_sticky_mask():
    """A {0,-inf} sticky mask restricts the derivations (constituency.py:280-289)."""
    need_gpu()
    root, rules, emis = batch_pcfg(6000, 1, 6, 3, 3)
    sticky = np.zeros((1, 6, 6))
    sticky[0, 1, 3] = NEG_INF
    logz, marg, st = K.pcfg_fb(dev(root), dev(rules), dev(emis), dev(sticky))
    z, g = O.pcfg_gradients(root[0], rules[0], emis[0], sticky[0])
    assert abs(logz[0].item() - z) <= RTOL * abs(z)
    np.testing.assert_allclose(marg[0].cpu().numpy(), g["sticky"], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("case", [c for c in load("pcfg") if not c.vacuous], ids=lambda c: str(c.meta))
def test_pcfg_golden_gradients_and_argmax(case):
    """potential_marginals returns all four gradients (dist.py:113-114);
    argmax is bit-exact (fp64 max-plus, first-max walk)."""
    need_gpu()
    x = inputs(case)
    d = sd.PCFG(x["root"], x["binary_rules"], x["emissions"])
    pm = sd.potential_marginals(d)
    assert sorted(pm) == ["binary_rules", "emissions", "root", "sticky"]
    for k in pm:
        if f"pmarg_{k}" in case or f"pmarg_{k}_idx" in case:
            case.check_marg(k, pm[k], RTOL, ATOL, prefix="pmarg_")
    ind, score, algo = sd.argmax_info(d)
    assert algo == "max-plus-pcfg"
    np.testing.assert_array_equal(ind["sticky"], case["argmax_sticky"])
    assert score == float(case.argmax_score)


@pytest.mark.parametrize("B,n,nt,pt", [(3, 12, 5, 7), (2, 2, 3, 2), (2, 24, 32, 17), (2, 9, 1, 1)])
def test_pcfg_gradients_vs_oracle(B, n, nt, pt):
    need_gpu()
    root, rules, emis = batch_pcfg(4100, B, n, nt, pt)
    logz, g, st = K.pcfg_grad(dev(root), dev(rules), dev(emis))
    assert (st.cpu().numpy() == 0).all()
    for b in range(B):
        z, go = O.pcfg_gradients(root[b], rules[b], emis[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z) + 1e-9
        for k in ("root", "binary_rules", "emissions", "sticky"):
            np.testing.assert_allclose(g[k][b].cpu().numpy(), go[k], rtol=RTOL, atol=ATOL, err_msg=k)


@pytest.mark.parametrize("B,n,nt,pt", [(3, 12, 5, 7), (2, 20, 8, 8), (2, 1, 3, 2), (2, 16, 32, 32)])
def test_pcfg_argmax_vs_oracle(B, n, nt, pt):
    need_gpu()
    root, rules, emis = batch_pcfg(4200, B, n, nt, pt)
    mask, score, st = K.pcfg_viterbi(dev(root), dev(rules), dev(emis))
    for b in range(B):
        if n == 1:
            assert st[b].item() == 1
            continue
        mo, so = O.pcfg_argmax(root[b], rules[b], emis[b])
        np.testing.assert_array_equal(mask[b].cpu().numpy(), mo)  # bit-exact
        assert score[b].item() == so


def test_pcfg_gradient_invariants_config():
    """C5b shape (B=128, n=64, NT=PT=32): expected rule counts sum to n-1
    binary nodes, root gradient to 1, each word's emission gradient to 1."""
    need_gpu()
    root, rules, emis = batch_pcfg(5100, 128, 64, 32, 32)
    logz, g, st = K.pcfg_grad(dev(root), dev(rules), dev(emis))
    assert (st == 0).all()
    gd = {k: v.double() for k, v in g.items()}
    one = torch.ones(128, dtype=torch.float64, device="cuda")
    assert torch.allclose(gd["root"].sum(1), one, rtol=1e-4)
    assert torch.allclose(gd["binary_rules"].sum((1, 2, 3)), 63 * one, rtol=1e-4)
    assert torch.allclose(gd["emissions"].sum(2), torch.ones(128, 64, dtype=torch.float64, device="cuda"), rtol=1e-4)
    assert torch.allclose(gd["sticky"].sum((1, 2)), 127 * one, rtol=1e-4)


def test_pcfg_log_prob_masked_inside():
    """dist.py:266-271: log-prob of a bracketing via the masked inside; the
    argmax bracketing has the highest probability among a few random ones."""
    need_gpu()
    root, rules, emis = batch_pcfg(4300, 1, 10, 6, 5)
    d = sd.PCFG(root[0], rules[0], emis[0])
    ind = sd.argmax(d)
    lp, algo = sd.log_prob_info(d, ind)
    assert algo == "pcfg-masked-inside"
    n = 10
    mask = np.full((n, n), NEG_INF)
    for i, j in np.argwhere(ind["sticky"] > 0):
        mask[i, j] = 0.0
    zm = O.pcfg_log_partition(root[0], rules[0], emis[0], sticky=mask)
    z = O.pcfg_log_partition(root[0], rules[0], emis[0])
    assert abs(lp - (zm - z)) <= 1e-4 * max(1.0, abs(zm - z))
    bad = dict(ind)
    bad["sticky"] = ind["sticky"].copy()
    bad["sticky"][0, 0] = 0.0
    with pytest.raises(sd.InvalidProblem):
        sd.log_prob(d, bad)


@pytest.mark.parametrize("B,n,nt,pt", [(2, 8, 40, 36), (2, 70, 3, 2), (1, 6, 64, 96), (2, 5, 33, 1)])
def test_pcfg_general_shapes_vs_oracle(B, n, nt, pt):
    """Grammars / sentences outside the fast kernel's shape (n > 64 or NT, PT >
    32: the paper's NT=64, PT=96 grammar) run on the general
    fp64 inside-outside kernel (pcfg_gen.cu): log Z, span marginals, all four
    gradients and the argmax against the oracle."""
    need_gpu()
    root, rules, emis = batch_pcfg(4300, B, n, nt, pt)
    logz, marg, st = K.pcfg_fb(dev(root), dev(rules), dev(emis))
    gl, g, st2 = K.pcfg_grad(dev(root), dev(rules), dev(emis))
    assert (st.cpu().numpy() == 0).all() and (st2.cpu().numpy() == 0).all()
    for b in range(B):
        z, go = O.pcfg_gradients(root[b], rules[b], emis[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z) + 1e-9
        assert abs(gl[b].item() - z) <= RTOL * abs(z) + 1e-9
        np.testing.assert_allclose(marg[b].cpu().numpy(), go["sticky"], rtol=RTOL, atol=ATOL)
        for k in ("root", "binary_rules", "emissions", "sticky"):
            np.testing.assert_allclose(g[k][b].cpu().numpy(), go[k], rtol=RTOL, atol=ATOL, err_msg=k)
    if n <= 12:
        mask, score, st3 = K.pcfg_viterbi(dev(root), dev(rules), dev(emis))
        for b in range(B):
            mo, so = O.pcfg_argmax(root[b], rules[b], emis[b])
            np.testing.assert_array_equal(mask[b].cpu().numpy(), mo)
            assert score[b].item() == so


def test_pcfg_paper_grammar_api():
    """The drop-in API at the paper's PCFG grammar size (NT=64, PT=96) with a
    sticky span mask: log_partition / marginals / log_prob run (general path)."""
    need_gpu()
    root, rules, emis = batch_pcfg(4400, 1, 6, 64, 96)
    d = sd.PCFG(root[0], rules[0], emis[0])
    z = sd.log_partition(d)
    zo = O.pcfg_log_partition(root[0], rules[0], emis[0])
    assert abs(z - zo) <= RTOL * abs(zo)
    m = sd.marginals(d)["sticky"]
    np.testing.assert_allclose(m, O.pcfg_gradients(root[0], rules[0], emis[0])[1]["sticky"], rtol=RTOL, atol=ATOL)
    ind = sd.argmax(d)
    lp = sd.log_prob(d, ind)
    assert lp <= 0.0 and np.isfinite(lp)
