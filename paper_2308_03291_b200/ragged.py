"""Inference-neutral padding so that instances of different lengths share
ONE kernel launch (the reference's own notion is
`pad_chain`, chain.py:161-176: padded steps carry the log-space identity, so
every structure extends uniquely and log Z / the marginals of the original
parts are unchanged).

Per family, `key` groups instances that can share a launch, `size` is the
ragged extent, `pad(d, size)` builds the padded instance and `unpad(d, x)`
slices a marginal / indicator dict back to `d`'s shape:

* LinearChainCRF: identity transitions appended (chain.py:161-176);
* MonotoneAlignmentCRF: a forced corridor (n,m) -> (N,m) -> (N,M) of zero
  DOWN / RIGHT moves, every other padded move -inf;
* CTCDist: blank-only frames PREPENDED (blank potential 0, other labels
  -inf): every original lattice path is extended by exactly one all-blank
  prefix, and the first original frame sees the same alpha;
* SpanningTreeCRF, multi-root only: extra nodes whose ONLY arc is root -> node
  (weight exp(0) = 1; no outgoing arcs), projective-compatible since they sit
  after position n;
* SemiMarkovCRF: width-1 identity segments appended (label kept, potential 0;
  every other padded segment, and every original segment that would now run
  past position n, -inf): each labelled segmentation extends uniquely;
* TreeCRF: the padded words are single-word spans (label 0, potential 0) and
  the only spans that cover them are the left-branching (0, j), j >= n (label
  0, potential 0); every other span touching a padded word is -inf, so every
  binary tree over the n words extends by exactly one tree;
* PCFG: the grammar gains a nonterminal X and a preterminal P (every
  instance of the group, so the shapes agree).  A padded word emits only P;
  X is the new start symbol (root[X] = 0) with rules X -> X P and
  X -> A P (A an original nonterminal, weight root[A]), each times 1/2 so
  X's rules stay normalised; the only derivations are the original ones
  extended left-branching over the padded words, so the span marginals are
  unchanged and log Z drops by exactly (N - n) log 2 (`logz_shift`).

Host-side glue only: the padded batch runs through the same kernels.
"""

from __future__ import annotations

import numpy as np

from .families import (CTCDist, LinearChainCRF, MonotoneAlignmentCRF, PCFG, SemiMarkovCRF, SpanningTreeCRF,
                       TreeCRF)

NEG_INF = float("-inf")


def _chain_pad(d, n):
    extra = n - d.n
    if extra == 0:
        return d
    pad = np.full((extra, d.m, d.m), NEG_INF)
    idx = np.arange(d.m)
    pad[:, idx, idx] = 0.0
    return LinearChainCRF(d.init, np.concatenate([d.transitions, pad], axis=0))


def _chain_unpad(d, x):
    return {"init": x["init"], "transitions": x["transitions"][: d.n - 1]}


def _nw_pad(d, size):
    N, M = size
    if (N, M) == (d.n, d.m):
        return d
    th = np.full((N + 1, M + 1, 3), NEG_INF)
    th[: d.n + 1, : d.m + 1] = d.move_potentials
    th[d.n + 1:, d.m, 1] = 0.0        # DOWN along column m
    th[N, d.m + 1:, 2] = 0.0          # RIGHT along row N
    return MonotoneAlignmentCRF(th)


def _nw_unpad(d, x):
    return {"move_potentials": x["move_potentials"][: d.n + 1, : d.m + 1]}


def _ctc_pad(d, T):
    extra = T - d.num_frames
    if extra == 0:
        return d
    pad = np.full((extra, d.vocab_size), NEG_INF)
    pad[:, 0] = 0.0  # BLANK = 0 (alignment.py:195)
    return CTCDist(np.concatenate([pad, d.frame_potentials], axis=0), d.target)


def _ctc_unpad(d, x):
    return {"frame_potentials": x["frame_potentials"][-d.num_frames:]}


def _span_pad(d, n):
    extra = n - d.n
    if extra == 0:
        return d
    adj = np.full((n + 1, n + 1), NEG_INF)
    adj[: d.n + 1, : d.n + 1] = d.adjacency
    adj[0, d.n + 1:] = 0.0
    return SpanningTreeCRF(adj, directed=d.directed, projective=d.projective, single_root_edge=False)


def _span_unpad(d, x):
    return {"adjacency": x["adjacency"][: d.n + 1, : d.n + 1]}


def _sm_pad(d, n):
    th0 = d.segment_potentials
    n0, s, m, _ = th0.shape
    if n == n0:
        return d
    th = np.full((n, s, m, m), NEG_INF)
    th[:n0] = th0
    for w in range(1, s + 1):  # original segments that would now end past n0
        th[max(n0 - w + 1, 0):n0, w - 1] = NEG_INF
    idx = np.arange(m)
    th[n0:, 0, idx, idx] = 0.0
    return SemiMarkovCRF(th)


def _sm_unpad(d, x):
    return {"segment_potentials": x["segment_potentials"][: d.segment_potentials.shape[0]]}


def _tree_pad(d, n):
    th0 = d.span_potentials
    n0, _, m = th0.shape
    if n == n0:
        return d
    th = np.full((n, n, m), NEG_INF)
    th[:n0, :n0] = th0
    k = np.arange(n0, n)
    th[k, k, 0] = 0.0      # padded words
    th[0, n0:, 0] = 0.0    # (0, j), j >= n0: the original tree, then one padded word at a time
    return TreeCRF(th)


def _tree_unpad(d, x):
    n0 = d.span_potentials.shape[0]
    return {"span_potentials": x["span_potentials"][:n0, :n0]}


LOG_HALF = -float(np.log(2.0))


def _pcfg_pad(d, n):
    nt0, pt0, n0 = d.num_nt, d.num_pt, d.n
    nt, pt = nt0 + 1, pt0 + 1
    X, P = nt0, nt + pt0  # X: new nonterminal; P: new preterminal (child index)
    cmap = np.concatenate([np.arange(nt0), nt + np.arange(pt0)])  # original child -> new child index
    rules = np.full((nt, nt + pt, nt + pt), NEG_INF)
    rules[np.ix_(np.arange(nt0), cmap, cmap)] = d.binary_rules
    rules[X, X, P] = LOG_HALF
    rules[X, np.arange(nt0), P] = d.root + LOG_HALF
    root = np.full(nt, NEG_INF)
    if n > n0:
        root[X] = 0.0
    else:
        root[:nt0] = d.root
    emis = np.full((n, pt), NEG_INF)
    emis[:n0, :pt0] = d.emissions
    emis[n0:, pt0] = 0.0
    sticky = np.zeros((n, n))
    sticky[:n0, :n0] = d.sticky
    return PCFG(root, rules, emis, sticky)


def _pcfg_unpad(d, x):
    return {"sticky": x["sticky"][: d.n, : d.n]}


def logz_shift(d, padded) -> float:
    """log Z(d) - log Z(padded) (0 except for the PCFG's 1/2 per padded word)."""
    if isinstance(d, PCFG):
        return (padded.n - d.n) * float(np.log(2.0))
    return 0.0


# family -> (key, size, combine sizes, pad, unpad)
RAGGED = {
    LinearChainCRF: (lambda d: (d.m,), lambda d: d.n, max, _chain_pad, _chain_unpad),
    MonotoneAlignmentCRF: (lambda d: (), lambda d: (d.n, d.m),
                           lambda ss: (max(s[0] for s in ss), max(s[1] for s in ss)), _nw_pad, _nw_unpad),
    CTCDist: (lambda d: (d.vocab_size, len(d.target)), lambda d: d.num_frames, max, _ctc_pad, _ctc_unpad),
    SpanningTreeCRF: (lambda d: (d.directed, d.projective), lambda d: d.n, max, _span_pad, _span_unpad),
    SemiMarkovCRF: (lambda d: d.segment_potentials.shape[1:3], lambda d: d.segment_potentials.shape[0], max,
                    _sm_pad, _sm_unpad),
    TreeCRF: (lambda d: (d.span_potentials.shape[2],), lambda d: d.span_potentials.shape[0], max,
              _tree_pad, _tree_unpad),
    PCFG: (lambda d: (d.num_nt, d.num_pt), lambda d: d.n, max, _pcfg_pad, _pcfg_unpad),
}


def raggable(d) -> bool:
    if type(d) not in RAGGED:
        return False
    return not (isinstance(d, SpanningTreeCRF) and d.single_root_edge)


def group_key(d):
    return (type(d), RAGGED[type(d)][0](d))


def native_ragged(ds) -> bool:
    """Groups the kernels serve WITHOUT padding, through per-instance lengths
    (chains: sdb_chain_fb_lengths / sdb_chain_viterbi_lengths)."""
    if not isinstance(ds[0], LinearChainCRF) or not needs_padding(ds):
        return False
    from . import backends
    from .kernels import chain_ragged_supported

    if backends.exact_now():  # the exact-mode chain kernel takes same-length groups (padded instead)
        return False
    from .dist import _large, _tiny

    if _large(ds) or _tiny(ds):  # such a group runs in the exact mode (dist._run): padded as well
        return False

    return chain_ragged_supported(max(d.n for d in ds), ds[0].m)


def needs_padding(ds) -> bool:
    _, size, _, _, _ = RAGGED[type(ds[0])]
    return len({size(d) for d in ds}) > 1


def pad_fits(ds) -> bool:
    """Can the padded group run on the kernels?  The PCFG padding adds one
    nonterminal and one preterminal (kernels.PCFG_MAX_NT / _PT bound them)."""
    if isinstance(ds[0], PCFG):
        from .kernels import PCFG_MAX_NT, PCFG_MAX_PT

        return ds[0].num_nt + 1 <= PCFG_MAX_NT and ds[0].num_pt + 1 <= PCFG_MAX_PT
    return True


def pad_group(ds):
    """-> padded instances (all the same shape); a group whose instances
    already share their length is returned unchanged."""
    _, size, comb, pad, _ = RAGGED[type(ds[0])]
    if not needs_padding(ds):
        return list(ds)
    target = comb([size(d) for d in ds])
    return [pad(d, target) for d in ds]


def unpad(d, x):
    return RAGGED[type(d)][4](d, x)
