"""Ragged batches on the GPU: instances of different lengths share ONE
launch per group through inference-neutral padding and match the
per-instance results (log Z, marginals, argmax)."""

import numpy as np
import torch
import pytest

import paper_2308_03291_b200 as sd
from golden.builders import alignment, chain, ctc, pcfg, semi_markov, spanning, tree
from gpu_util import ATOL, RTOL, need_gpu

pytestmark = pytest.mark.gpu


def _check(dists):
    lz = sd.batch_map(sd.log_partition, dists)
    mg = sd.batch_map(sd.marginals, dists)
    for d, z, m in zip(dists, lz, mg):
        z0 = sd.log_partition(d)
        assert abs(z - z0) <= RTOL * abs(z0) + 1e-6
        m0 = sd.marginals(d)
        for k in m0:
            assert m[k].shape == m0[k].shape
            np.testing.assert_allclose(m[k], m0[k], rtol=RTOL, atol=ATOL)


def test_ragged_chains():
    need_gpu()
    dists = [sd.LinearChainCRF(*chain(s, n, 5)) for s, n in enumerate([3, 17, 40, 1, 9])]
    _check(dists)
    am = sd.batch_map(sd.argmax_info, dists)
    for d, (ind, score, algo) in zip(dists, am):
        ind0, score0, _ = sd.argmax_info(d)
        for k in ind0:
            np.testing.assert_array_equal(ind[k], ind0[k])
        assert score == score0


def test_ragged_alignments():
    need_gpu()
    dists = [sd.MonotoneAlignmentCRF(alignment(s, n, m)) for s, (n, m) in enumerate([(5, 7), (40, 12), (12, 30), (1, 1)])]
    _check(dists)


def test_ragged_ctc_and_spanning():
    need_gpu()
    dists = [sd.CTCDist(*ctc(s, T, 6, 3)) for s, T in enumerate([7, 19, 30])]
    _check(dists)
    for proj in (False, True):
        dists = [sd.SpanningTreeCRF(spanning(s, n, True), projective=proj) for s, n in enumerate([3, 11, 20])]
        _check(dists)


def test_ragged_semimarkov_and_tree():
    need_gpu()
    dists = [sd.SemiMarkovCRF(semi_markov(s, n, 3, 4)) for s, n in enumerate([3, 11, 25, 7])]
    _check(dists)
    dists = [sd.TreeCRF(tree(s, n, 3)) for s, n in enumerate([1, 6, 19, 12])]
    _check(dists)
    for dists in ([sd.SemiMarkovCRF(semi_markov(s, n, 3, 4)) for s, n in enumerate([3, 11, 25])],
                  [sd.TreeCRF(tree(s, n, 3)) for s, n in enumerate([2, 9, 17])]):
        am = sd.batch_map(sd.argmax_info, dists)
        for d, (ind, score, algo) in zip(dists, am):
            ind0, score0, algo0 = sd.argmax_info(d)
            for k in ind0:
                np.testing.assert_array_equal(ind[k], ind0[k])
            assert score == score0 and algo == algo0


def test_ragged_pcfg():
    """PCFGs of different lengths (same NT, PT) share one launch through the
    X -> X P / X -> A P padding grammar; log Z, span marginals and the best
    derivation (score less the padding's log 2 per padded word) match."""
    need_gpu()
    dists = [sd.PCFG(*pcfg(s, n, 3, 2)) for s, n in enumerate([2, 7, 12, 5])]
    _check(dists)
    am = sd.batch_map(sd.argmax_info, dists)
    for d, (ind, score, algo) in zip(dists, am):
        ind0, score0, algo0 = sd.argmax_info(d)
        np.testing.assert_array_equal(ind["sticky"], ind0["sticky"])
        assert abs(score - score0) <= 1e-4 * abs(score0) and algo == algo0


def test_batch_map_pcfg_full_grammar():
    """NT = PT = 32 (the C5b grammar): same-length groups run unpadded and
    ragged groups whose padded grammar would not fit the kernel run as
    exact-shape groups -- no NativeError."""
    need_gpu()
    same = [sd.PCFG(*pcfg(40 + s, 10, 32, 32)) for s in range(3)]
    got = sd.batch_map(sd.log_partition, same)
    for d, z in zip(same, got):
        assert abs(z - sd.log_partition(d)) <= 1e-5 * abs(z)
    mixed = [sd.PCFG(*pcfg(50 + s, n, 32, 32)) for s, n in enumerate([6, 9, 6])]
    got = sd.batch_map(sd.marginals, mixed)
    for d, m in zip(mixed, got):
        np.testing.assert_allclose(m["sticky"], sd.marginals(d)["sticky"], rtol=1e-5, atol=1e-7)


def test_ragged_chain_native_lengths():
    """Chains of different lengths run through the per-instance-length kernels
    (no padding compute): log Z, marginals and Viterbi equal the per-instance
    calls; the kernel zeroes marginals / tags past each instance's length."""
    need_gpu()
    from paper_2308_03291_b200 import kernels as K
    from paper_2308_03291_b200 import ragged as rg

    # m = 12: not every instance is below dist.AUTO_EXACT_SIZE, so the group stays on the fp32 ragged kernels
    dists = [sd.LinearChainCRF(*chain(70 + s, n, 12)) for s, n in enumerate([3, 40, 17, 1, 64, 2])]
    assert rg.native_ragged(dists)
    _check(dists)
    am = sd.batch_map(sd.argmax_info, dists)
    for d, (ind, score, algo) in zip(dists, am):
        ind0, score0, algo0 = sd.argmax_info(d)
        for k in ind0:
            np.testing.assert_array_equal(ind[k], ind0[k])
        assert score == score0 and algo == algo0
    # raw kernel contract: zeros past the length
    init = torch.stack([torch.as_tensor(d.init, dtype=torch.float32) for d in dists]).cuda()
    tr = torch.zeros(len(dists), 63, 12, 12)
    for i, d in enumerate(dists):
        tr[i, : d.n - 1] = torch.as_tensor(d.transitions, dtype=torch.float32)
    lens = torch.tensor([d.n for d in dists], dtype=torch.int32).cuda()
    lz, mi, mt, st = K.chain_fb(init, tr.cuda(), True, lens)
    tags, score, st2 = K.chain_viterbi(init, tr.cuda(), lens)
    for i, d in enumerate(dists):
        assert (mt[i, d.n - 1:] == 0).all() and (tags[i, d.n:] == 0).all()
