"""Inference-neutral padding for ragged batches (paper_2308_03291_b200/ragged.py),
checked on the CPU oracle: log Z unchanged and the original parts'
marginals unchanged after padding (chain.py:161-176, test_chain.py:58-62)."""

import numpy as np
import pytest

from golden.builders import alignment, chain, ctc, pcfg, semi_markov, spanning, tree
from oracle import sd_oracle as O
from paper_2308_03291_b200 import ragged as rg
from paper_2308_03291_b200.families import (PCFG, CTCDist, LinearChainCRF, MonotoneAlignmentCRF, SemiMarkovCRF,
                                             SpanningTreeCRF, TreeCRF)


def test_chain_padding_neutral():
    init, tr = chain(11, 4, 3)
    d = LinearChainCRF(init, tr)
    p = rg._chain_pad(d, 7)
    assert p.n == 7
    z0, mi0, mt0 = O.chain_marginals(d.init[None], d.transitions[None])
    z1, mi1, mt1 = O.chain_marginals(p.init[None], p.transitions[None])
    assert abs(z0[0] - z1[0]) <= 1e-9
    u = rg.unpad(d, {"init": mi1[0], "transitions": mt1[0]})
    np.testing.assert_allclose(u["transitions"], mt0[0], atol=1e-12)


@pytest.mark.parametrize("size", [(9, 6), (5, 11), (9, 11)])
def test_alignment_padding_neutral(size):
    d = MonotoneAlignmentCRF(alignment(3, 5, 6))
    p = rg._nw_pad(d, size)
    z0, m0 = O.nw_marginals(d.move_potentials)
    z1, m1 = O.nw_marginals(p.move_potentials)
    assert abs(z0 - z1) <= 1e-9
    np.testing.assert_allclose(rg.unpad(d, {"move_potentials": m1})["move_potentials"], m0, atol=1e-12)
    # the argmax path extends through the corridor
    mask0, s0 = O.nw_argmax(d.move_potentials)
    mask1, s1 = O.nw_argmax(p.move_potentials)
    assert s0 == s1
    np.testing.assert_array_equal(rg.unpad(d, {"move_potentials": mask1})["move_potentials"], mask0)


def test_ctc_padding_neutral():
    fp, tg = ctc(4, 9, 5, 3)
    d = CTCDist(fp, tg)
    p = rg._ctc_pad(d, 14)
    z0, m0 = O.ctc_marginals(fp[None], np.asarray(tg)[None])
    z1, m1 = O.ctc_marginals(p.frame_potentials[None], np.asarray(tg)[None])
    assert abs(z0[0] - z1[0]) <= 1e-9
    np.testing.assert_allclose(rg.unpad(d, {"frame_potentials": m1[0]})["frame_potentials"], m0[0], atol=1e-12)


@pytest.mark.parametrize("projective", [False, True])
def test_spanning_multiroot_padding_neutral(projective):
    adj = spanning(5, 6, True)
    d = SpanningTreeCRF(adj, directed=True, projective=projective)
    p = rg._span_pad(d, 9)
    if projective:
        z0, m0 = O.eisner_marginals(adj)
        z1, m1 = O.eisner_marginals(p.adjacency)
    else:
        z0, m0 = O.mtt_log_partition(adj), O.mtt_marginals(adj)
        z1, m1 = O.mtt_log_partition(p.adjacency), O.mtt_marginals(p.adjacency)
    assert abs(z0 - z1) <= 1e-9
    np.testing.assert_allclose(rg.unpad(d, {"adjacency": m1})["adjacency"], m0, atol=1e-9)


@pytest.mark.parametrize("n0,n", [(5, 9), (1, 4), (6, 6)])
def test_semimarkov_padding_neutral(n0, n):
    d = SemiMarkovCRF(semi_markov(12, n0, min(3, n0), 3))
    p = rg._sm_pad(d, n)
    assert p.segment_potentials.shape[0] == n
    z0, m0 = O.sm_marginals(d.segment_potentials)
    z1, m1 = O.sm_marginals(p.segment_potentials)
    assert abs(z0 - z1) <= 1e-9
    np.testing.assert_allclose(rg.unpad(d, {"segment_potentials": m1})["segment_potentials"], m0, atol=1e-12)
    seg0, s0 = O.sm_viterbi(d.segment_potentials)
    seg1, s1 = O.sm_viterbi(p.segment_potentials)
    assert s0 == s1
    assert [g for g in seg1 if g[0] < n0] == [g for g in seg0]


@pytest.mark.parametrize("n0,n", [(5, 9), (1, 3), (7, 8)])
def test_tree_padding_neutral(n0, n):
    d = TreeCRF(tree(13, n0, 3))
    p = rg._tree_pad(d, n)
    z0, m0 = O.tree_marginals(d.span_potentials)
    z1, m1 = O.tree_marginals(p.span_potentials)
    assert abs(z0 - z1) <= 1e-9
    np.testing.assert_allclose(rg.unpad(d, {"span_potentials": m1})["span_potentials"], m0, atol=1e-12)
    lab0, s0 = O.tree_argmax(d.span_potentials)
    lab1, s1 = O.tree_argmax(p.span_potentials)
    assert s0 == s1
    np.testing.assert_array_equal(lab1[:n0, :n0], lab0)


@pytest.mark.parametrize("n0,n", [(4, 7), (1, 3), (5, 5)])
def test_pcfg_padding_neutral(n0, n):
    d = PCFG(*pcfg(14, n0, 3, 2))
    p = rg._pcfg_pad(d, n)
    assert (p.num_nt, p.num_pt, p.n) == (4, 3, n)
    args0 = (d.root, d.binary_rules, d.emissions, d.sticky)
    args1 = (p.root, p.binary_rules, p.emissions, p.sticky)
    z0, z1 = O.pcfg_log_partition(*args0), O.pcfg_log_partition(*args1)
    if z0 == -np.inf:  # one word: no binary derivation (vacuous) on both sides
        assert z1 == -np.inf
        return
    assert abs(z0 - (z1 + rg.logz_shift(d, p))) <= 1e-9
    m0, m1 = O.pcfg_span_marginals(*args0), O.pcfg_span_marginals(*args1)
    m0 = m0[1] if isinstance(m0, tuple) else m0
    m1 = m1[1] if isinstance(m1, tuple) else m1
    np.testing.assert_allclose(rg.unpad(d, {"sticky": m1})["sticky"], m0, atol=1e-12)
    a0, s0 = O.pcfg_argmax(*args0)
    a1, s1 = O.pcfg_argmax(*args1)
    np.testing.assert_array_equal(np.asarray(a1)[:n0, :n0], a0)
    assert abs(s0 - (s1 + rg.logz_shift(d, p))) <= 1e-9


def test_groups():
    a = LinearChainCRF(*chain(1, 3, 2))
    b = LinearChainCRF(*chain(2, 8, 2))
    c = LinearChainCRF(*chain(3, 5, 4))
    assert rg.group_key(a) == rg.group_key(b) != rg.group_key(c)
    assert not rg.raggable(SpanningTreeCRF(spanning(1, 3, True), single_root_edge=True))
    pa, pb = rg.pad_group([a, b])
    assert pa.n == pb.n == 8


def test_pad_group_same_length_is_identity():
    """A group whose instances share their length is not padded (the PCFG
    pad would otherwise add a nonterminal and a preterminal)."""
    ds = [PCFG(*pcfg(s, 5, 3, 2)) for s in range(3)]
    assert all(a is b for a, b in zip(rg.pad_group(ds), ds))
    assert not rg.needs_padding(ds)
    full = [PCFG(*pcfg(s, n, 32, 32)) for s, n in enumerate([4, 6])]
    assert rg.needs_padding(full) and not rg.pad_fits(full)
