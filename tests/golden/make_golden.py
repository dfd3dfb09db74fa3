"""Generate golden vectors by running the UNMODIFIED reference (`structdist`
0.1.0 under /root/reference/pkg/src) on seeded, float32-rounded inputs.

Run in the build container (the reference does not exist on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden_<family>.npz.  Each case stores its inputs (small
cases) or its seed + shape (scale cases, rebuilt by builders.py), the
reference's log_partition, marginals (or a fixed subsample of entries plus
full-array sums for the large ones), and the argmax indicator + score.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import builders as bld  # noqa: E402
import structdist as sd  # noqa: E402
from structdist.dist import potential_marginals  # noqa: E402

NEG_INF = float("-inf")
SUBSAMPLE = 4096


class Store:
    def __init__(self):
        self.arrays = {}
        self.meta = []

    def add(self, fam, meta, **arrays):
        idx = len(self.meta)
        meta = dict(meta, idx=idx, family=fam)
        self.meta.append(meta)
        for k, v in arrays.items():
            self.arrays[f"c{idx:03d}__{k}"] = np.asarray(v)


def _sub_idx(size, seed=0):
    rng = np.random.default_rng(10_000 + seed)
    if size <= SUBSAMPLE:
        return np.arange(size)
    return np.sort(rng.choice(size, SUBSAMPLE, replace=False))


def run(dist, store, fam, meta, inputs, big=False, argmax=True, pot_marg=False):
    out = {}
    out["logz"] = np.array(sd.log_partition(dist))
    try:
        marg = sd.marginals(dist)
        out["vacuous"] = np.array(0)
        for k, v in marg.items():
            if big:
                flat = v.ravel()
                ix = _sub_idx(flat.size, meta.get("seed", 0))
                out[f"marg_{k}_idx"] = ix
                out[f"marg_{k}_val"] = flat[ix]
                out[f"marg_{k}_sum"] = np.array(flat.sum())
            else:
                out[f"marg_{k}"] = v
    except sd.VacuousDistribution:
        out["vacuous"] = np.array(1)
    if pot_marg and not out["vacuous"]:
        for k, v in potential_marginals(dist).items():
            out[f"pmarg_{k}"] = v
    if argmax and not out["vacuous"]:
        try:
            ind, score, algo = sd.argmax_info(dist)
            for k, v in ind.items():
                out[f"argmax_{k}"] = v.astype(np.int8) if big else v
            out["argmax_score"] = np.array(score)
            meta = dict(meta, argmax_algo=algo)
        except sd.VacuousDistribution:
            out["argmax_vacuous"] = np.array(1)
    if not big:
        for k, v in inputs.items():
            out[f"in_{k}"] = v
    store.add(fam, meta, **out)


def chain_cases(st):
    for seed, (n, m) in enumerate([(1, 2), (2, 2), (3, 3), (4, 2), (5, 3), (6, 2), (8, 5), (17, 7), (33, 4)]):
        init, tr = bld.chain(seed, n, m)
        run(sd.LinearChainCRF(init, tr), st, "chain", dict(seed=seed, n=n, m=m), dict(init=init, transitions=tr))
    # closed forms / forbidden / vacuous (test_chain.py:15-26, test_dist_ops.py:249-258)
    run(sd.LinearChainCRF(np.zeros(2), np.zeros((2, 2, 2))), st, "chain", dict(kind="zeros"),
        dict(init=np.zeros(2), transitions=np.zeros((2, 2, 2))))
    tr = np.zeros((1, 2, 2)); tr[0, :, 1] = NEG_INF
    run(sd.LinearChainCRF(np.zeros(2), tr), st, "chain", dict(kind="forbidden"), dict(init=np.zeros(2), transitions=tr))
    tr = np.full((2, 2, 2), NEG_INF)
    run(sd.LinearChainCRF(np.zeros(2), tr), st, "chain", dict(kind="vacuous"), dict(init=np.zeros(2), transitions=tr))
    tr = np.zeros((1, 2, 2)); tr[0] = [[0.0, 5.0], [1.0, 0.0]]
    run(sd.LinearChainCRF(np.zeros(2), tr), st, "chain", dict(kind="viterbi5"), dict(init=np.zeros(2), transitions=tr))
    # config-scale instance (C1 shape): n=128, m=32
    init, tr = bld.chain(0, 128, 32)
    run(sd.LinearChainCRF(init, tr), st, "chain", dict(seed=0, n=128, m=32, scale=1), {}, big=True)


def semi_markov_cases(st):
    for seed, (n, s, m) in enumerate([(1, 1, 2), (2, 2, 1), (4, 2, 2), (5, 3, 2), (6, 4, 3), (9, 3, 4), (16, 5, 3)]):
        th = bld.semi_markov(seed, n, s, m)
        run(sd.SemiMarkovCRF(th), st, "semi_markov", dict(seed=seed, n=n, s=s, m=m), dict(segment_potentials=th))
    run(sd.SemiMarkovCRF(np.zeros((3, 3, 1, 1))), st, "semi_markov", dict(kind="zeros"),
        dict(segment_potentials=np.zeros((3, 3, 1, 1))))
    th = bld.semi_markov(7, 64, 8, 32)
    run(sd.SemiMarkovCRF(th), st, "semi_markov", dict(seed=7, n=64, s=8, m=32, scale=1), {}, big=True)


def alignment_cases(st):
    for seed, (n, m) in enumerate([(1, 1), (1, 3), (2, 3), (3, 3), (4, 2), (5, 7), (9, 4), (16, 16)]):
        mv = bld.alignment(seed, n, m)
        run(sd.MonotoneAlignmentCRF(mv), st, "alignment", dict(seed=seed, n=n, m=m), dict(move_potentials=mv))
    for n, m in [(1, 1), (2, 2), (3, 3)]:  # Delannoy 3, 13, 63
        mv = bld.zero_alignment(n, m)
        run(sd.MonotoneAlignmentCRF(mv), st, "alignment", dict(kind="zeros", n=n, m=m), dict(move_potentials=mv))
    mv = bld.alignment(5, 64, 32)
    run(sd.MonotoneAlignmentCRF(mv), st, "alignment", dict(seed=5, n=64, m=32, scale=1), {}, big=True)


def ctc_cases(st):
    for seed, (T, V, L) in enumerate([(1, 2, 1), (2, 2, 1), (4, 3, 2), (5, 3, 2), (6, 4, 3), (8, 5, 3), (12, 6, 4), (20, 9, 6)]):
        fp, tg = bld.ctc(seed, T, V, L)
        run(sd.CTCDist(fp, tg), st, "ctc", dict(seed=seed, T=T, V=V, L=L), dict(frame_potentials=fp, target=np.array(tg)))
    run(sd.CTCDist(np.zeros((2, 2)), (1,)), st, "ctc", dict(kind="zeros"),
        dict(frame_potentials=np.zeros((2, 2)), target=np.array([1])))
    # repeated label needs a blank in between; infeasible when too few frames
    run(sd.CTCDist(np.zeros((2, 3)), (1, 1)), st, "ctc", dict(kind="infeasible"),
        dict(frame_potentials=np.zeros((2, 3)), target=np.array([1, 1])))
    fp, tg = bld.ctc(11, 3, 3, 2)
    run(sd.CTCDist(fp, (2, 2)), st, "ctc", dict(kind="repeat"), dict(frame_potentials=fp, target=np.array([2, 2])))
    fp, tg = bld.ctc(9, 96, 32, 24)
    run(sd.CTCDist(fp, tg), st, "ctc", dict(seed=9, T=96, V=32, L=24, scale=1), dict(target=np.array(tg)), big=True)


def tree_cases(st):
    for seed, (n, m) in enumerate([(1, 1), (1, 3), (2, 2), (3, 2), (4, 1), (5, 3), (7, 2), (12, 4)]):
        th = bld.tree(seed, n, m)
        run(sd.TreeCRF(th), st, "tree", dict(seed=seed, n=n, m=m), dict(span_potentials=th))
    run(sd.TreeCRF(np.zeros((4, 4, 1))), st, "tree", dict(kind="zeros"), dict(span_potentials=np.zeros((4, 4, 1))))
    th = bld.tree(3, 64, 32)
    run(sd.TreeCRF(th), st, "tree", dict(seed=3, n=64, m=32, scale=1), {}, big=True)


def pcfg_cases(st):
    for seed, (n, nt, pt) in enumerate([(1, 1, 1), (2, 2, 2), (3, 2, 2), (3, 3, 2), (4, 2, 3), (5, 3, 3), (7, 4, 4), (10, 6, 5)]):
        root, rules, emis = bld.pcfg(seed, n, nt, pt)
        run(sd.PCFG(root, rules, emis), st, "pcfg", dict(seed=seed, n=n, nt=nt, pt=pt),
            dict(root=root, binary_rules=rules, emissions=emis), pot_marg=True)
    root, rules, emis = bld.pcfg(21, 14, 8, 8)
    run(sd.PCFG(root, rules, emis), st, "pcfg", dict(seed=21, n=14, nt=8, pt=8, scale=1),
        dict(root=root, binary_rules=rules, emissions=emis))


def spanning_cases(st):
    for directed in (True, False):
        for projective in (True, False):
            for single in (True, False):
                for seed, n in enumerate([1, 2, 3, 4, 5, 7]):
                    adj = bld.spanning(100 * seed + 7, n, directed)
                    d = sd.SpanningTreeCRF(adj, directed=directed, projective=projective, single_root_edge=single)
                    run(d, st, "spanning", dict(seed=100 * seed + 7, n=n, directed=directed, projective=projective,
                                                single=single), dict(adjacency=adj))
                adj = bld.zero_spanning(4)
                d = sd.SpanningTreeCRF(adj, directed=directed, projective=projective, single_root_edge=single)
                run(d, st, "spanning", dict(kind="zeros", n=4, directed=directed, projective=projective, single=single),
                    dict(adjacency=adj))
    adj = np.full((4, 4), NEG_INF)
    run(sd.SpanningTreeCRF(adj), st, "spanning", dict(kind="vacuous", n=3, directed=True, projective=False, single=False),
        dict(adjacency=adj), argmax=False)
    # exactly singular Laplacians with every column finite: a 2-cycle cut off from the root, and
    # (single root only) two root branches with no arc between them (numerics.py:143-146)
    cut = bld.spanning(41, 6)
    cut[:5, 5:] = NEG_INF
    cut[5:, :5] = NEG_INF
    cut[5, 6] = 0.3
    cut[6, 5] = -0.2
    br = np.full((5, 5), NEG_INF)
    br[0, 1] = 0.1; br[0, 2] = -0.4; br[1, 3] = 0.7; br[2, 4] = 0.2; br[3, 1] = 0.5
    for kind, adj in (("cutoff", cut), ("branches", br)):
        for single in (False, True):
            d = sd.SpanningTreeCRF(adj, directed=True, projective=False, single_root_edge=single)
            run(d, st, "spanning", dict(kind=kind, n=adj.shape[0] - 1, directed=True, projective=False, single=single),
                dict(adjacency=adj), argmax=False)
    for projective in (False, True):
        for single in (False, True):
            n = 128 if not projective else 64
            adj = bld.spanning(2000 + n + single, n)
            d = sd.SpanningTreeCRF(adj, directed=True, projective=projective, single_root_edge=single)
            run(d, st, "spanning", dict(seed=2000 + n + single, n=n, directed=True, projective=projective,
                                        single=single, scale=1), {}, big=True, argmax=projective)


def sample_cases(st):
    """Reference samples (dist.py:179-212, one seeded stream, num=2) for the
    families the GPU samples: chain FFBS, alignment, CTC, Tree-CRF and
    projective spanning trees (Eisner decode with Gumbel picks), plus the
    Eisner max-plus decode (spanning.py:323-325)."""
    from structdist.spanning import eisner_max_arcs  # noqa: E402

    def add(fam, d, meta, inputs):
        inds, algo = sd.sample_info(d, meta["seed"], num=2)
        out = {f"in_{k}": v for k, v in inputs.items()}
        for r, ind in enumerate(inds):
            for k, v in ind.items():
                out[f"sample{r}_{k}"] = v
        st.add(fam, dict(meta, algo=algo), **out)

    for seed, (n, m) in enumerate([(1, 3), (2, 2), (5, 3), (12, 4), (30, 6)]):
        init, tr = bld.chain(seed, n, m)
        add("chain", sd.LinearChainCRF(init, tr), dict(seed=seed, n=n, m=m), dict(init=init, transitions=tr))
    for seed, (n, m) in enumerate([(1, 1), (3, 2), (6, 9), (20, 13)]):
        mv = bld.alignment(seed, n, m)
        add("alignment", sd.MonotoneAlignmentCRF(mv), dict(seed=seed, n=n, m=m), dict(move_potentials=mv))
    for seed, (T, V, L) in enumerate([(1, 2, 1), (5, 3, 2), (12, 6, 4), (30, 8, 9)]):
        fp, tg = bld.ctc(seed, T, V, L)
        add("ctc", sd.CTCDist(fp, tg), dict(seed=seed, T=T, V=V, L=L), dict(frame_potentials=fp, target=np.array(tg)))
    for seed, (n, m) in enumerate([(1, 2), (4, 3), (9, 2), (16, 5)]):
        th = bld.tree(seed, n, m)
        add("tree", sd.TreeCRF(th), dict(seed=seed, n=n, m=m), dict(span_potentials=th))
    for single in (False, True):
        for seed, n in enumerate([1, 3, 6, 11]):
            adj = bld.spanning(300 + seed, n, True)
            d = sd.SpanningTreeCRF(adj, directed=True, projective=True, single_root_edge=single)
            add("spanning", d, dict(seed=seed, n=n, single=single), dict(adjacency=adj))
            arcs = eisner_max_arcs(d)
            mx = np.zeros_like(adj)
            for h, dd in arcs:
                mx[h, dd] = 1.0
            st.arrays[f"c{len(st.meta) - 1:03d}__eisner_max"] = mx


def wilson_cases(st):
    """Reference Wilson samples (non-projective, spanning.py:517-558)."""
    for single in (False, True):
        for seed, n in enumerate([2, 5, 9, 16]):
            adj = bld.spanning(500 + seed, n, True)
            d = sd.SpanningTreeCRF(adj, directed=True, projective=False, single_root_edge=single)
            inds, algo = sd.sample_info(d, seed, num=2)
            out = {"in_adjacency": adj}
            for r, ind in enumerate(inds):
                out[f"sample{r}_adjacency"] = ind["adjacency"]
            st.add("spanning", dict(seed=seed, n=n, single=single, algo=algo), **out)


def colbourn_cases(st):
    """Reference Colbourn samples (sequential conditioning on Matrix-Tree
    marginals, spanning.py:567-603), num=2 from one stream; the point-mass
    case of test_spanning.py:180-189."""
    for single in (False, True):
        for seed, n in enumerate([2, 5, 9, 16, 24]):
            adj = bld.spanning(600 + seed, n, True)
            d = sd.SpanningTreeCRF(adj, directed=True, projective=False, single_root_edge=single)
            inds, algo = sd.sample_info(d, seed, num=2, algorithm="colbourn")
            out = {"in_adjacency": adj}
            for r, ind in enumerate(inds):
                out[f"sample{r}_adjacency"] = ind["adjacency"]
            st.add("spanning", dict(seed=seed, n=n, single=single, algo=algo), **out)
    adj = np.full((4, 4), NEG_INF)
    adj[0, 1] = adj[1, 2] = adj[2, 3] = 0.0
    for seed in range(3):
        inds, algo = sd.sample_info(sd.SpanningTreeCRF(adj, directed=True), seed, num=2, algorithm="colbourn")
        out = {"in_adjacency": adj}
        for r, ind in enumerate(inds):
            out[f"sample{r}_adjacency"] = ind["adjacency"]
        st.add("spanning", dict(seed=seed, n=3, single=False, algo=algo, kind="point_mass"), **out)


def sample2_cases(st):
    """Reference samples for the semi-Markov CRF and the PCFG (chain.py:330-344,
    constituency.py:374-378), num=2 from one stream."""
    for seed, (n, sw, m) in enumerate([(1, 1, 2), (6, 3, 2), (12, 4, 3)]):
        th = bld.semi_markov(seed, n, sw, m)
        inds, algo = sd.sample_info(sd.SemiMarkovCRF(th), seed, num=2)
        out = {"in_segment_potentials": th}
        for r, ind in enumerate(inds):
            out[f"sample{r}_segment_potentials"] = ind["segment_potentials"]
        st.add("semi_markov", dict(seed=seed, n=n, s=sw, m=m, algo=algo), **out)
    for seed, (n, nt, pt) in enumerate([(2, 2, 2), (5, 3, 2), (8, 4, 4)]):
        root, rules, emis = bld.pcfg(seed, n, nt, pt)
        inds, algo = sd.sample_info(sd.PCFG(root, rules, emis), seed, num=2)
        out = {"in_root": root, "in_binary_rules": rules, "in_emissions": emis}
        for r, ind in enumerate(inds):
            out[f"sample{r}_sticky"] = ind["sticky"]
        st.add("pcfg", dict(seed=seed, n=n, nt=nt, pt=pt, algo=algo), **out)



# ----------------------------------------------------------- derived ops

DERIVED_SHAPES = {
    "chain": [dict(n=1, m=3), dict(n=5, m=3), dict(n=24, m=6)],
    "semi_markov": [dict(n=4, s=2, m=2), dict(n=9, s=3, m=3)],
    "alignment": [dict(n=3, m=2), dict(n=12, m=9)],
    "ctc": [dict(T=6, V=4, L=3), dict(T=20, V=7, L=6)],
    "tree": [dict(n=1, m=2), dict(n=5, m=3), dict(n=12, m=4)],
    "pcfg": [dict(n=3, nt=2, pt=2), dict(n=6, nt=3, pt=3)],
    "spanning": [dict(n=n, directed=dr, projective=pr, single=sg)
                 for n in (3, 6) for dr in (True, False) for pr in (True, False) for sg in (True, False)],
}


def _bad_indicators(fam, d, good):
    """Structurally invalid indicators derived from a valid one (each must
    raise InvalidProblem in the reference's validate_indicator)."""
    bad = []
    z = {k: np.zeros_like(v) for k, v in good.items()}
    bad.append(z)                                             # marks nothing
    k0 = next(iter(good))
    half = {k: v.copy() for k, v in good.items()}
    half[k0] = half[k0] * 0.5
    bad.append(half)                                          # not 0/1
    if fam == "chain":
        two = {k: v.copy() for k, v in good.items()}
        two["init"][:] = 1.0                                  # two initial tags
        bad.append(two)
        if d.n > 2:
            dis = {k: v.copy() for k, v in good.items()}
            t = dis["transitions"][1]
            a, b = np.argwhere(t > 0)[0]
            t[a, b] = 0.0
            t[(a + 1) % d.m, b] = 1.0                         # disconnected at step 1
            bad.append(dis)
    elif fam == "semi_markov":
        gap = {k: v.copy() for k, v in good.items()}
        hot = np.argwhere(gap["segment_potentials"] > 0)
        gap["segment_potentials"][tuple(hot[-1])] = 0.0       # no longer covers n
        bad.append(gap)
    elif fam == "alignment":
        off = {k: v.copy() for k, v in good.items()}
        mv = off["move_potentials"]
        cells = np.argwhere(mv.sum(axis=2) == 0)
        i, j = cells[len(cells) // 2]
        mv[i, j, 0 if (i > 0 and j > 0) else (1 if i > 0 else 2)] = 1.0  # a move off the path
        bad.append(off)
    elif fam == "ctc":
        blank = {k: v.copy() for k, v in good.items()}
        blank["frame_potentials"][:] = 0.0
        blank["frame_potentials"][:, 0] = 1.0                 # all blanks: collapses to ()
        bad.append(blank)
    elif fam == "tree" and d.n > 1:
        br = {k: v.copy() for k, v in good.items()}
        sp = br["span_potentials"]
        sp[0, d.n - 1] = 0.0                                  # root span missing
        sp[1, d.n - 1, 0] = 1.0 if sp[1, d.n - 1].sum() == 0 else sp[1, d.n - 1, 0]
        bad.append(br)
        two = {k: v.copy() for k, v in good.items()}
        two["span_potentials"][0, 0, :] = 1.0                 # a span with several labels
        bad.append(two)
    elif fam == "pcfg":
        br = {k: v.copy() for k, v in good.items()}
        br["sticky"][0, d.n - 1] = 0.0
        bad.append(br)
    elif fam == "spanning":
        adj = good["adjacency"]
        n = d.n
        two = {"adjacency": adj.copy()}
        dep = int(np.argwhere(adj > 0)[0][1])
        h = [x for x in range(n + 1) if x != dep and adj[x, dep] == 0][0]
        two["adjacency"][h, dep] = 1.0                        # two heads
        bad.append(two)
        if n >= 3:
            cyc = {"adjacency": np.zeros_like(adj)}
            cyc["adjacency"][0, 1] = 1.0
            for c in range(2, n + 1):
                cyc["adjacency"][c + 1 if c < n else 2, c] = 1.0  # 2 -> n -> n-1 ... cycle
            bad.append(cyc)
            star = {"adjacency": np.zeros_like(adj)}
            star["adjacency"][0, 1:] = 1.0                    # every node on the root
            bad.append(star)                                  # invalid only with single_root_edge
            cross = {"adjacency": np.zeros_like(adj)}
            cross["adjacency"][0, 1] = 1.0
            cross["adjacency"][1, 3] = 1.0
            cross["adjacency"][3, 2] = 1.0
            for c in range(4, n + 1):
                cross["adjacency"][3, c] = 1.0
            cross["adjacency"][0, 2] = 0.0
            bad.append(cross)                                 # 1->3 and 3->2 fine; crossing below
            cr2 = {"adjacency": np.zeros_like(adj)}
            cr2["adjacency"][0, 2] = 1.0
            cr2["adjacency"][2, 1] = 1.0
            cr2["adjacency"][1, 3] = 1.0                      # 1->3 crosses 0->2
            for c in range(4, n + 1):
                cr2["adjacency"][3, c] = 1.0
            bad.append(cr2)
    shp = {k: np.zeros(tuple(s + 1 for s in v.shape)) for k, v in good.items()}
    bad.append(shp)                                           # wrong shape
    return bad


def derived_cases(st):
    """entropy / cross_entropy / kl_divergence (dist.py:306-347) and log_prob
    with validate_indicator (dist.py:224-276) from the unmodified reference."""
    for fam, shapes in DERIVED_SHAPES.items():
        for si, shape in enumerate(shapes):
            seed = 700 + 10 * si + len(st.meta)
            p_in = bld.family_inputs(fam, seed, shape)
            q_in = bld.family_inputs(fam, seed + 1, shape)
            if fam == "ctc":
                q_in["target"] = p_in["target"]
            if fam == "spanning" and not shape["directed"]:
                pass
            p = bld.make_dist(sd, fam, p_in, shape)
            q = bld.make_dist(sd, fam, q_in, shape)
            out = {f"in_{k}": v for k, v in p_in.items()}
            out.update({f"q_{k}": v for k, v in q_in.items()})
            h_p, algo = sd.dist.entropy_info(p)
            out["entropy_p"] = np.array(h_p)
            out["cross_pq"] = np.array(sd.cross_entropy(p, q))
            out["kl_pq"] = np.array(sd.kl_divergence(p, q))
            good, _, _ = sd.argmax_info(p)
            out["logprob_argmax"] = np.array(sd.log_prob(p, good))
            smp = sd.sample(p, seed)
            for k, v in smp.items():
                out[f"sample_{k}"] = v
            out["logprob_sample"] = np.array(sd.log_prob(p, smp))
            bads = _bad_indicators(fam, p, good)
            raises = []
            for b, ind in enumerate(bads):
                for k, v in ind.items():
                    out[f"bad{b}_{k}"] = v
                try:
                    raises.append(float(sd.log_prob(p, ind)))
                except sd.InvalidProblem:
                    raises.append(np.nan)  # NaN marks "raised InvalidProblem"
            out["bad_logprob"] = np.array(raises)
            st.add(fam, dict(shape, seed=seed, algo=algo, nbad=len(bads)), **out)
    # support mismatch -> +inf cross-entropy; point mass -> entropy 0 (test_dist_ops.py:144-194)
    init, tr = bld.chain(900, 4, 3)
    tq = tr.copy()
    tq[1, :, 2] = NEG_INF
    p, q = sd.LinearChainCRF(init, tr), sd.LinearChainCRF(init, tq)
    st.add("chain", dict(kind="support", n=4, m=3, nbad=0), in_init=init, in_transitions=tr, q_init=init,
           q_transitions=tq, entropy_p=np.array(sd.entropy(p)), cross_pq=np.array(sd.cross_entropy(p, q)),
           kl_pq=np.array(sd.kl_divergence(p, q)))
    tpm = np.full((3, 3, 3), NEG_INF)
    for t in range(3):
        tpm[t, t % 3, (t + 1) % 3] = 0.5
    ipm = np.array([0.0, NEG_INF, NEG_INF])
    p = sd.LinearChainCRF(ipm, tpm)
    st.add("chain", dict(kind="point_mass", n=4, m=3, nbad=0), in_init=ipm, in_transitions=tpm, q_init=ipm,
           q_transitions=tpm, entropy_p=np.array(sd.entropy(p)), cross_pq=np.array(sd.cross_entropy(p, p)),
           kl_pq=np.array(sd.kl_divergence(p, p)))

def main():
    fams = {
        "chain": chain_cases, "semi_markov": semi_markov_cases, "alignment": alignment_cases,
        "ctc": ctc_cases, "tree": tree_cases, "pcfg": pcfg_cases, "spanning": spanning_cases,
        "sample": sample_cases, "wilson": wilson_cases, "sample2": sample2_cases,
        "colbourn": colbourn_cases, "derived": derived_cases,
    }
    only = sys.argv[1:] or list(fams)
    for fam in only:
        t0 = time.time()
        st = Store()
        fams[fam](st)
        st.arrays["meta_json"] = np.array(json.dumps(st.meta))
        path = os.path.join(HERE, f"golden_{fam}.npz")
        np.savez_compressed(path, **st.arrays)
        print(f"{fam}: {len(st.meta)} cases, {os.path.getsize(path)/1e3:.0f} kB, {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
