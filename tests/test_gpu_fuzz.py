"""Seeded shape / mask fuzzing of every family's batched kernels against the
float64 oracle: random sizes (including the size classes where the dispatch
switches kernels), random forbidden entries (-inf), vacuous instances mixed
into the batch.  log Z and marginals at the parity bar, argmax bit-exact."""

import numpy as np
import pytest
import torch

from paper_2308_03291_b200 import kernels as K
from gpu_util import ATOL, NEG_INF, RTOL, dev, need_gpu
from golden.builders import (batch_alignment, batch_chain, batch_ctc, batch_pcfg, batch_semi_markov, batch_spanning,
                             batch_tree)
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


def _mask(rng, x, p, keep=None):
    """Forbid a random fraction p of the entries (never the `keep` boolean mask)."""
    m = rng.random(x.shape) < p
    if keep is not None:
        m &= ~keep
    x = x.copy()
    x[m] = NEG_INF
    return x


def _check_lz(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    assert np.array_equal(np.isneginf(got), np.isneginf(want)), (got, want)
    f = ~np.isneginf(want)
    np.testing.assert_allclose(got[f], want[f], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_chain(seed):
    need_gpu()
    rng = np.random.default_rng(100 + seed)
    B, n, m = int(rng.integers(1, 5)), int(rng.choice([1, 2, 5, 17, 40, 130])), int(rng.choice([2, 7, 32, 33]))
    init, tr = batch_chain(200 + seed, B, n, m)
    tr = _mask(rng, tr, 0.2)
    logz, mi, mt, st = K.chain_fb(dev(init), dev(tr))
    z, pi, pt = O.chain_marginals(init, tr)
    _check_lz(logz.cpu(), z)
    np.testing.assert_allclose(mt.cpu().numpy(), pt, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(mi.cpu().numpy(), pi, rtol=RTOL, atol=ATOL)
    tags, score, st2 = K.chain_viterbi(dev(init), dev(tr))
    ot, os_ = O.chain_viterbi(init, tr)
    ok = ~np.isneginf(z)
    np.testing.assert_array_equal(tags.cpu().numpy()[ok], ot[ok])
    np.testing.assert_array_equal(score.cpu().numpy()[ok], os_[ok])


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_alignment(seed):
    need_gpu()
    rng = np.random.default_rng(300 + seed)
    n = int(rng.choice([1, 3, 40, 160, 300]))
    m = int(rng.choice([1, 5, 31, 32, 64, 96, 129, 360]))
    B = 2
    th = batch_alignment(400 + seed, B, n, m)
    keep = np.zeros(th.shape[1:], dtype=bool)
    th = np.stack([_mask(rng, t, 0.1) for t in th])
    logz, marg, st = K.nw_fb(dev(th))
    path, score, st2 = K.nw_viterbi(dev(th))
    for b in range(B):
        z, mg = O.nw_marginals(th[b])
        _check_lz([logz[b].item()], [z])
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        if z > NEG_INF:
            mask, sc = O.nw_argmax(th[b])
            p = path[b].cpu().numpy()
            got = np.zeros_like(mask)
            ii, jj = np.nonzero(p >= 0)
            got[ii, jj, p[ii, jj]] = 1
            np.testing.assert_array_equal(got, mask)
            assert score[b].item() == sc
    del keep


@pytest.mark.parametrize("seed", range(10))
def test_fuzz_ctc(seed):
    need_gpu()
    rng = np.random.default_rng(500 + seed)
    T, V, L = int(rng.choice([1, 6, 30, 90])), int(rng.choice([2, 5, 40])), int(rng.choice([0, 1, 3, 12]))
    fp, tg = batch_ctc(600 + seed, 3, T, V, L)
    fp = np.stack([_mask(rng, f, 0.1) for f in fp])
    logz, marg, st = K.ctc_fb(dev(fp), dev(tg, torch.int32))
    z, mg = O.ctc_marginals(fp, tg)
    _check_lz(logz.cpu(), z)
    np.testing.assert_allclose(marg.cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
    labs, score, _ = K.ctc_viterbi(dev(fp), dev(tg, torch.int32))
    ol, os_ = O.ctc_argmax(fp, tg)
    ok = ~np.isneginf(z)
    np.testing.assert_array_equal(labs.cpu().numpy()[ok], ol[ok])
    np.testing.assert_array_equal(score.cpu().numpy()[ok], os_[ok])


@pytest.mark.parametrize("seed", range(10))
def test_fuzz_tree(seed):
    need_gpu()
    rng = np.random.default_rng(700 + seed)
    n, m = int(rng.choice([1, 2, 9, 33, 64, 129])), int(rng.choice([1, 3, 8]))
    th = batch_tree(800 + seed, 2, n, m)
    th = np.stack([_mask(rng, t, 0.15) for t in th])
    logz, marg, st = K.tree_fb(dev(th))
    labels, score, st2 = K.tree_viterbi(dev(th))
    for b in range(2):
        z, mg = O.tree_marginals(th[b])
        _check_lz([logz[b].item()], [z])
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        if z > NEG_INF:
            lab, sc = O.tree_argmax(th[b])
            np.testing.assert_array_equal(labels[b].cpu().numpy(), lab)
            assert score[b].item() == sc


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("single", [False, True])
def test_fuzz_spanning(seed, single):
    need_gpu()
    rng = np.random.default_rng(900 + seed + 50 * single)
    n = int(rng.choice([1, 2, 6, 40, 128, 140]))
    adj = batch_spanning(1000 + seed, 2, n)
    eye = np.eye(n + 1, dtype=bool)
    adj = np.stack([_mask(rng, a, 0.2, keep=eye) for a in adj])
    for b in range(2):
        adj[b][:, 0] = NEG_INF
        np.fill_diagonal(adj[b], NEG_INF)
    lz, mg, st = K.mtt(dev(adj), single)
    le, me, se = K.eisner(dev(adj), single)
    heads, _, sk = K.kuhlmann(dev(adj), single)
    for b in range(2):
        z = O.mtt_log_partition(adj[b], single)
        _check_lz([lz[b].item()], [z])
        if z > NEG_INF:
            np.testing.assert_allclose(mg[b].cpu().numpy(), O.mtt_marginals(adj[b], single), rtol=RTOL, atol=ATOL)
        ze = O.eisner_log_partition(adj[b], single)
        _check_lz([le[b].item()], [ze])
        if ze > NEG_INF:
            em = O.eisner_marginals(adj[b], single)
            em = em[1] if isinstance(em, tuple) else em
            np.testing.assert_allclose(me[b].cpu().numpy(), em, rtol=RTOL, atol=ATOL)
            kh = O.kuhlmann_heads(adj[b], single)
            if kh is not None:
                np.testing.assert_array_equal(heads[b].cpu().numpy(), kh)


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_semi_markov(seed):
    need_gpu()
    rng = np.random.default_rng(1100 + seed)
    n, s_, m = int(rng.choice([1, 4, 30])), int(rng.choice([1, 3, 8])), int(rng.choice([1, 4, 16]))
    s_ = min(s_, n)  # the family requires 1 <= s <= n (chain.py:232-233)
    th = batch_semi_markov(1200 + seed, 2, n, s_, m)
    th = np.stack([_mask(rng, t, 0.2) for t in th])
    logz, marg, st = K.semimarkov_fb(dev(th))
    for b in range(2):
        z, mg = O.sm_marginals(th[b])
        _check_lz([logz[b].item()], [z])
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_pcfg(seed):
    need_gpu()
    rng = np.random.default_rng(1300 + seed)
    n, nt, pt = int(rng.choice([1, 2, 7, 20])), int(rng.choice([1, 3, 32, 40])), int(rng.choice([1, 4, 32]))
    r, ru, e = batch_pcfg(1400 + seed, 2, n, nt, pt)
    st_mask = np.zeros((2, n, n))
    st_mask[rng.random((2, n, n)) < 0.1] = NEG_INF  # forbidden brackets through the sticky channel
    logz, marg, st = K.pcfg_fb(dev(r), dev(ru), dev(e), dev(st_mask))
    for b in range(2):
        z, g = O.pcfg_gradients(r[b], ru[b], e[b], st_mask[b])
        _check_lz([logz[b].item()], [z])
        want = g["sticky"] if g is not None else np.zeros((n, n))  # vacuous: zero marginals
        np.testing.assert_allclose(marg[b].cpu().numpy(), want, rtol=RTOL, atol=ATOL)
