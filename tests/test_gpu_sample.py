"""GPU sampling parity (dist.py:179-212): same seed -> the same structures
as the reference (golden_sample.npz, num=2 from one stream) and as the
oracle's per-pick Gumbel draws at larger sizes; Eisner max-plus decode
(spanning.py:323-325) bit-exact."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import dev, need_gpu
from golden.builders import batch_alignment, batch_chain, batch_ctc, batch_spanning, batch_tree
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu
CASES = load("sample")


def _dist(case):
    x = inputs(case)
    fam = case.meta["family"]
    if fam == "chain":
        return sd.LinearChainCRF(x["init"], x["transitions"])
    if fam == "alignment":
        return sd.MonotoneAlignmentCRF(x["move_potentials"])
    if fam == "ctc":
        return sd.CTCDist(x["frame_potentials"], tuple(int(v) for v in np.atleast_1d(x["target"])))
    if fam == "tree":
        return sd.TreeCRF(x["span_potentials"])
    return sd.SpanningTreeCRF(x["adjacency"], directed=True, projective=True, single_root_edge=bool(case.meta["single"]))


@pytest.mark.parametrize("case", CASES, ids=lambda c: str(c.meta))
def test_sample_golden(case):
    need_gpu()
    d = _dist(case)
    inds, algo = sd.sample_info(d, int(case.meta["seed"]), num=2)
    assert algo == case.meta["algo"]
    for r, ind in enumerate(inds):
        for k, v in ind.items():
            np.testing.assert_array_equal(v, case[f"sample{r}_{k}"], err_msg=f"sample {r} {k}")
    if case.meta["family"] == "spanning":  # eisner_max_arcs
        heads, _, st = K.eisner_decode(dev(case["in_adjacency"][None]), bool(case.meta["single"]))
        h = heads[0, 0].cpu().numpy()
        mask = np.zeros_like(case["in_adjacency"])
        mask[h[1:], np.arange(1, len(h))] = 1
        np.testing.assert_array_equal(mask, case["eisner_max"])


def _seeds(B):
    return [31 + 7 * b for b in range(B)]


def test_chain_sample_vs_oracle():
    need_gpu()
    B, n, m, num = 4, 64, 16, 3
    init, tr = batch_chain(70, B, n, m)
    noise = torch.stack([torch.as_tensor(np.random.default_rng(s).gumbel(size=num * n * m)) for s in _seeds(B)]).cuda()
    tags, used, st = K.chain_sample(dev(init), dev(tr), noise, num)
    assert (st == 0).all() and (used == num * n * m).all()
    for b, s in enumerate(_seeds(B)):
        rng = np.random.default_rng(s)
        for r in range(num):
            np.testing.assert_array_equal(tags[b, r].cpu().numpy(), O.chain_sample(init[b], tr[b], rng))


def test_alignment_sample_vs_oracle():
    need_gpu()
    B, n, m, num = 3, 60, 40, 2
    th = batch_alignment(71, B, n, m)
    cnt = K.stream_len("alignment", dict(n=n, m=m))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(s).gumbel(size=num * cnt)) for s in _seeds(B)]).cuda()
    path, used, st = K.nw_sample(dev(th), noise, num)
    assert (st == 0).all()
    for b, s in enumerate(_seeds(B)):
        rng = np.random.default_rng(s)
        for r in range(num):
            np.testing.assert_array_equal(path[b, r].cpu().numpy(), O.nw_sample(th[b], rng))


def test_ctc_sample_vs_oracle():
    need_gpu()
    B, T, V, L, num = 3, 80, 12, 20, 2
    fp, tg = batch_ctc(72, B, T, V, L)
    cnt = K.stream_len("ctc", dict(T=T))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(s).gumbel(size=num * cnt)) for s in _seeds(B)]).cuda()
    states, used, st = K.ctc_sample(dev(fp), torch.as_tensor(tg, dtype=torch.int32).cuda(), noise, num)
    assert (st == 0).all()
    for b, s in enumerate(_seeds(B)):
        rng = np.random.default_rng(s)
        for r in range(num):
            np.testing.assert_array_equal(states[b, r].cpu().numpy(), O.ctc_sample(fp[b], tg[b], rng))


@pytest.mark.parametrize("n", [24, 140])  # 140: past the old 128-span walk stack
def test_tree_sample_vs_oracle(n):
    need_gpu()
    B, m, num = 3, 6, 2
    th = batch_tree(73, B, n, m)
    cnt = K.stream_len("tree", dict(n=n, m=m))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(s).gumbel(size=num * cnt)) for s in _seeds(B)]).cuda()
    labels, used, st = K.tree_sample(dev(th), noise, num)
    assert (st == 0).all()
    for b, s in enumerate(_seeds(B)):
        rng = np.random.default_rng(s)
        for r in range(num):
            np.testing.assert_array_equal(labels[b, r].cpu().numpy(), O.tree_sample(th[b], rng))


@pytest.mark.parametrize("n", [40, 150])
@pytest.mark.parametrize("single", [False, True])
def test_eisner_sample_and_max_decode_vs_oracle(single, n):
    need_gpu()
    B, num = 3, 2
    adj = batch_spanning(74, B, n)
    cnt = K.stream_len("eisner", dict(n=n))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(s).gumbel(size=num * cnt)) for s in _seeds(B)]).cuda()
    heads, used, st = K.eisner_decode(dev(adj), single, noise, num)
    assert (st == 0).all()
    hmax, _, _ = K.eisner_decode(dev(adj), single)
    for b, s in enumerate(_seeds(B)):
        rng = np.random.default_rng(s)
        for r in range(num):
            np.testing.assert_array_equal(heads[b, r].cpu().numpy(), O.eisner_sample(adj[b], single, rng))
        np.testing.assert_array_equal(hmax[b, 0].cpu().numpy(), O.eisner_decode(adj[b], single))


def test_sample_vacuous_and_unsupported():
    need_gpu()
    tr = np.full((2, 2, 2), -np.inf)
    with pytest.raises(sd.VacuousDistribution):
        sd.sample(sd.LinearChainCRF(np.zeros(2), tr), 0)
    with pytest.raises(sd.InvalidProblem):
        sd.sample_info(sd.LinearChainCRF(np.zeros(2), np.zeros((1, 2, 2))), 0, num=0)
    adj = batch_spanning(75, 1, 5)[0]
    with pytest.raises(sd.InvalidProblem):
        sd.sample_info(sd.SpanningTreeCRF(adj, projective=False), 0, algorithm="no-such-sampler")


@pytest.mark.parametrize("case", load("wilson"), ids=lambda c: str(c.meta))
def test_wilson_golden(case):
    """Non-projective sampling (Wilson, spanning.py:517-558): identical to the
    reference for the same seed (num=2 from one stream)."""
    need_gpu()
    d = sd.SpanningTreeCRF(case["in_adjacency"], directed=True, projective=False,
                           single_root_edge=bool(case.meta["single"]))
    inds, algo = sd.sample_info(d, int(case.meta["seed"]), num=2)
    assert algo == case.meta["algo"]
    for r, ind in enumerate(inds):
        np.testing.assert_array_equal(ind["adjacency"], case[f"sample{r}_adjacency"])


def test_wilson_vs_oracle_config_size():
    need_gpu()
    B, n = 4, 128
    adj = batch_spanning(76, B, n)
    streams = [K.GumbelStream(s) for s in _seeds(B)]
    parent, st = K.wilson(dev(adj), streams)
    assert (st == 0).all()
    for b, s in enumerate(_seeds(B)):
        np.testing.assert_array_equal(parent[b].cpu().numpy(), O.wilson_sample(adj[b], False, np.random.default_rng(s)))


@pytest.mark.parametrize("case", load("colbourn"), ids=lambda c: str(c.meta))
def test_colbourn_golden(case):
    """Colbourn's sequential conditioning (spanning.py:567-603): identical to
    the reference for the same seed (num=2 from one stream), incl. the
    point-mass case of test_spanning.py:180-189."""
    need_gpu()
    d = sd.SpanningTreeCRF(case["in_adjacency"], directed=True, projective=False,
                           single_root_edge=bool(case.meta["single"]))
    inds, algo = sd.sample_info(d, int(case.meta["seed"]), num=2, algorithm="colbourn")
    assert algo == case.meta["algo"]
    for r, ind in enumerate(inds):
        np.testing.assert_array_equal(ind["adjacency"], case[f"sample{r}_adjacency"])


@pytest.mark.parametrize("single", [False, True])
def test_colbourn_batched_vs_oracle(single):
    """Batched GPU Colbourn (one mtt launch per dependent for all instances)
    against the oracle's per-instance restatement, n=40."""
    from paper_2308_03291_b200.backends import SpanningBackend

    need_gpu()
    B, n = 3, 40
    adj = batch_spanning(77, B, n)
    ds = [sd.SpanningTreeCRF(adj[b], directed=True, projective=False, single_root_edge=single) for b in range(B)]
    seeds = [31 + b for b in range(B)]
    out, algo = SpanningBackend().sample(ds, seeds, 2, "colbourn")
    assert algo == "colbourn"
    for b in range(B):
        rng = np.random.default_rng(seeds[b])
        for r in range(2):
            heads, fell = O.colbourn_sample(adj[b], single, rng)
            assert not fell
            mask = np.zeros((n + 1, n + 1))
            mask[heads[1:], np.arange(1, n + 1)] = 1.0
            np.testing.assert_array_equal(out[b][r]["adjacency"], mask)


@pytest.mark.parametrize("single", [False, True])
def test_colbourn_fallback_vs_oracle(single, monkeypatch):
    """The degenerate-marginals branch (spanning.py:592-597): forcing the
    column test to fail at the first dependent on both sides, the GPU path
    must finish with Wilson walks on the same conditioned weights and the
    same stream position as the oracle, and report the fallback name."""
    from paper_2308_03291_b200.backends import SpanningBackend

    need_gpu()
    monkeypatch.setattr(SpanningBackend, "COLBOURN_COL_TOL", -1.0)
    monkeypatch.setattr(O, "COLBOURN_COL_TOL", -1.0)
    B, n = 2, 24
    adj = batch_spanning(79, B, n)
    ds = [sd.SpanningTreeCRF(adj[b], directed=True, projective=False, single_root_edge=single) for b in range(B)]
    seeds = [41, 42]
    out, algo = SpanningBackend().sample(ds, seeds, 2, "colbourn")
    assert algo == "colbourn+wilson-fallback"
    for b in range(B):
        rng = np.random.default_rng(seeds[b])
        for r in range(2):
            heads, fell = O.colbourn_sample(adj[b], single, rng)
            assert fell
            mask = np.zeros((n + 1, n + 1))
            mask[heads[1:], np.arange(1, n + 1)] = 1.0
            np.testing.assert_array_equal(out[b][r]["adjacency"], mask)


def test_colbourn_wilson_agree_in_distribution():
    """Both exact samplers target the same distribution: on a 3-node problem
    (16 trees) the empirical tree frequencies of 300 Colbourn and 300 Wilson
    draws agree with the exact Matrix-Tree probabilities (loose tolerance)."""
    need_gpu()
    adj = batch_spanning(78, 1, 3)[0]
    d = sd.SpanningTreeCRF(adj, directed=True, projective=False)
    lz = float(sd.log_partition(d))
    counts = {}
    for algo in ("colbourn", "wilson"):
        inds, _ = sd.sample_info(d, 5, num=300, algorithm=algo)
        for ind in inds:
            key = (algo, tuple(np.argmax(ind["adjacency"][:, 1:], axis=0)))
            counts[key] = counts.get(key, 0) + 1
    for (algo, heads), c in counts.items():
        p = np.exp(sum(adj[h, dd + 1] for dd, h in enumerate(heads)) - lz)
        assert abs(c / 300 - p) < 0.1, (algo, heads, c, p)


@pytest.mark.parametrize("case", load("sample2"), ids=lambda c: str(c.meta))
def test_semimarkov_pcfg_sample_golden(case):
    need_gpu()
    x = inputs(case)
    if case.meta["family"] == "semi_markov":
        d, key = sd.SemiMarkovCRF(x["segment_potentials"]), "segment_potentials"
    else:
        d, key = sd.PCFG(x["root"], x["binary_rules"], x["emissions"]), "sticky"
    inds, algo = sd.sample_info(d, int(case.meta["seed"]), num=2)
    assert algo == case.meta["algo"]
    for r, ind in enumerate(inds):
        np.testing.assert_array_equal(ind[key], case[f"sample{r}_{key}"])


def test_semimarkov_pcfg_sample_vs_oracle():
    need_gpu()
    from golden.builders import batch_semi_markov, batch_pcfg
    B, n, s, m = 3, 40, 6, 8
    th = batch_semi_markov(77, B, n, s, m)
    cnt = K.stream_len("semi_markov", dict(n=n, s=s, m=m))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(x).gumbel(size=cnt)) for x in _seeds(B)]).cuda()
    seg, nseg, used, st = K.semimarkov_sample(dev(th), noise, 1)
    assert (st == 0).all()
    for b, x in enumerate(_seeds(B)):
        got = [tuple(v) for v in seg[b, 0, : nseg[b, 0]].cpu().numpy().tolist()]
        assert got == [tuple(int(z) for z in v) for v in O.sm_sample(th[b], np.random.default_rng(x))]
    B, n = 2, 12
    r, ru, e = batch_pcfg(78, B, n, 6, 5)
    cnt = K.stream_len("pcfg", dict(n=n, NT=6, PT=5))
    noise = torch.stack([torch.as_tensor(np.random.default_rng(x).gumbel(size=cnt)) for x in _seeds(B)]).cuda()
    mask, used, st = K.pcfg_sample(dev(r), dev(ru), dev(e), None, noise, 1)
    assert (st == 0).all()
    for b, x in enumerate(_seeds(B)):
        np.testing.assert_array_equal(mask[b, 0].cpu().numpy(), O.pcfg_sample(r[b], ru[b], e[b], np.random.default_rng(x)))
