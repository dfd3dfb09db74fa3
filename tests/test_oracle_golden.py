"""Pin the CPU oracle (oracle/sd_oracle.py) against the golden vectors the
unmodified reference produced (tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from golden_io import inputs, load
from oracle import sd_oracle as O

NEG_INF = float("-inf")


def _close(a, b, tol=1e-9):
    if b == NEG_INF:
        return a == NEG_INF
    return abs(a - b) <= tol * max(1.0, abs(b))


@pytest.mark.parametrize("case", load("chain"), ids=lambda c: str(c.meta))
def test_oracle_chain(case):
    x = inputs(case)
    init, tr = x["init"][None], x["transitions"][None]
    z, pi, pt = O.chain_marginals(init, tr)
    assert _close(z[0], float(case.logz))
    if not case.vacuous:
        case.check_marg("init", pi[0], rtol=1e-9, atol=1e-12)
        case.check_marg("transitions", pt[0], rtol=1e-9, atol=1e-12)
        tags, score = O.chain_viterbi(init, tr)
        ind_t = case["argmax_transitions"]
        m = init.shape[1]
        assert case["argmax_init"][tags[0, 0]] == 1
        for t in range(tr.shape[1]):
            assert ind_t[t, tags[0, t], tags[0, t + 1]] == 1
        assert _close(score[0], float(case.argmax_score))


@pytest.mark.parametrize("case", load("semi_markov"), ids=lambda c: str(c.meta))
def test_oracle_semi_markov(case):
    th = inputs(case)["segment_potentials"]
    z, marg = O.sm_marginals(th)
    assert _close(z, float(case.logz))
    case.check_marg("segment_potentials", marg, rtol=1e-9, atol=1e-12)
    segs, score = O.sm_viterbi(th)
    mask = np.zeros_like(th)
    for s0, w, p, l in segs:
        mask[s0, w - 1, p, l] = 1
    np.testing.assert_array_equal(mask, case["argmax_segment_potentials"])
    assert _close(score, float(case.argmax_score))


@pytest.mark.parametrize("case", load("alignment"), ids=lambda c: str(c.meta))
def test_oracle_alignment(case):
    th = inputs(case)["move_potentials"]
    z, marg = O.nw_marginals(th)
    assert _close(z, float(case.logz))
    case.check_marg("move_potentials", marg, rtol=1e-9, atol=1e-12)
    mask, score = O.nw_argmax(th)
    np.testing.assert_array_equal(mask, case["argmax_move_potentials"])
    assert _close(score, float(case.argmax_score))


@pytest.mark.parametrize("case", load("ctc"), ids=lambda c: str(c.meta))
def test_oracle_ctc(case):
    x = inputs(case)
    fp, tg = x["frame_potentials"][None], x["target"][None]
    z, marg = O.ctc_marginals(fp, tg)
    assert _close(z[0], float(case.logz))
    if not case.vacuous:
        case.check_marg("frame_potentials", marg[0], rtol=1e-9, atol=1e-12)
        labs, score = O.ctc_argmax(fp, tg)
        mask = np.zeros_like(fp[0])
        mask[np.arange(fp.shape[1]), labs[0]] = 1
        np.testing.assert_array_equal(mask, case["argmax_frame_potentials"])
        assert _close(score[0], float(case.argmax_score))


@pytest.mark.parametrize("case", load("tree"), ids=lambda c: str(c.meta))
def test_oracle_tree(case):
    th = inputs(case)["span_potentials"]
    z, marg = O.tree_marginals(th)
    assert _close(z, float(case.logz))
    case.check_marg("span_potentials", marg, rtol=1e-9, atol=1e-12)
    lab, score = O.tree_argmax(th)
    mask = np.zeros_like(th)
    ii, jj = np.nonzero(lab >= 0)
    mask[ii, jj, lab[ii, jj]] = 1
    np.testing.assert_array_equal(mask, case["argmax_span_potentials"])
    assert _close(score, float(case.argmax_score))


@pytest.mark.parametrize("case", load("pcfg"), ids=lambda c: str(c.meta))
def test_oracle_pcfg(case):
    x = inputs(case)
    z, grads = O.pcfg_gradients(x["root"], x["binary_rules"], x["emissions"])
    assert _close(z, float(case.logz))
    if case.vacuous:
        assert grads is None
        return
    case.check_marg("sticky", grads["sticky"], rtol=1e-9, atol=1e-12)
    # the split-batched restatement used as the C5b CPU baseline
    z2, span = O.pcfg_span_marginals(x["root"], x["binary_rules"], x["emissions"])
    assert _close(z2, float(case.logz))
    case.check_marg("sticky", span, rtol=1e-9, atol=1e-12)
    if "pmarg_binary_rules" in case:
        for k in ("root", "binary_rules", "emissions"):
            np.testing.assert_allclose(grads[k], case[f"pmarg_{k}"], rtol=1e-9, atol=1e-12)
    mask, score = O.pcfg_argmax(x["root"], x["binary_rules"], x["emissions"])
    np.testing.assert_array_equal(mask, case["argmax_sticky"])
    assert _close(score, float(case.argmax_score))


@pytest.mark.parametrize("case", load("spanning"), ids=lambda c: str(c.meta))
def test_oracle_spanning(case):
    m = case.meta
    adj = inputs(case)["adjacency"]
    single = m["single"]
    if m["projective"]:
        z = O.eisner_log_partition(adj, single)
        assert _close(z, float(case.logz))
        if not case.vacuous:
            z2, marg = O.eisner_marginals(adj, single)
            case.check_marg("adjacency", marg, rtol=1e-8, atol=1e-11)
            heads = O.kuhlmann_heads(adj, single)
            if "argmax_adjacency" in case:
                ind = np.asarray(case["argmax_adjacency"])
                want = np.full(adj.shape[0], -1)
                for h, d in zip(*np.nonzero(ind)):
                    want[d] = h
                np.testing.assert_array_equal(heads, want)
                # score computed the way dist.structure_score does
                assert _close(O.heads_score(adj, heads), float(case.argmax_score), 1e-12)
    else:
        z = O.mtt_log_partition(adj, single)
        assert _close(z, float(case.logz), 1e-8)
        if not case.vacuous:
            marg = O.mtt_marginals(adj, single)
            case.check_marg("adjacency", marg, rtol=1e-7, atol=1e-10)
            if "argmax_adjacency" in case:  # Chu-Liu-Edmonds (spanning.py:410-509)
                heads = O.cle_heads(adj, single)
                ind = np.asarray(case["argmax_adjacency"])
                want = np.full(adj.shape[0], -1)
                for h, d in zip(*np.nonzero(ind)):
                    want[d] = h
                np.testing.assert_array_equal(heads, want)
                assert _close(O.heads_score(adj, heads), float(case.argmax_score), 1e-12)


def test_oracle_closed_forms():
    # test_acceptance.py:54-66 style identities
    assert math.isclose(O.chain_log_partition(np.zeros((1, 2)), np.zeros((1, 2, 2, 2)))[0], 3 * math.log(2))
    _, ins = O.tree_inside(np.zeros((4, 4, 1)))
    assert math.isclose(ins[0, 3], math.log(5))
    assert math.isclose(O.sm_marginals(np.zeros((3, 3, 1, 1)))[0], math.log(4))
    assert math.isclose(O.ctc_log_partition(np.zeros((1, 2, 2)), np.array([[1]]))[0], math.log(3))
    adj = np.zeros((4, 4))
    adj[:, 0] = NEG_INF
    np.fill_diagonal(adj, NEG_INF)
    assert math.isclose(O.mtt_log_partition(adj), math.log(16))


def test_oracle_pcfg_span_marginals_sticky():
    """pcfg_span_marginals == pcfg_gradients' span marginals with a sticky
    (bracketing) mask, the masked-inside case (constituency.py:280-289)."""
    from golden import builders as bld

    r, ru, e = bld.pcfg(11, 8, 3, 4)
    stk = np.zeros((8, 8))
    stk[2, 5] = NEG_INF
    stk[0, 3] = NEG_INF
    z1, g = O.pcfg_gradients(r, ru, e, stk)
    z2, span = O.pcfg_span_marginals(r, ru, e, stk)
    assert _close(z1, z2)
    np.testing.assert_allclose(span, g["sticky"], rtol=1e-9, atol=1e-12)
