"""Host-side structure-indicator validation for `log_prob` (dist.py:224-248).

Restates the reference's per-family checks (same error class, same
conditions) so an indicator that does not encode exactly one structure of
the distribution raises `InvalidProblem` before any score is formed:

* chain        chain.py:141-158   (`indicator_to_tags`)
* semi-Markov  chain.py:356-372   (`indicator_to_segments`)
* alignment    alignment.py:170-187 (`validate_path_indicator`)
* CTC          alignment.py:357-364 (`validate_ctc_indicator`, `collapse` :346-354)
* Tree-CRF     constituency.py:143-176 (`is_binary_bracketing`, `validate_tree_indicator`)
* PCFG         constituency.py:381-386 (`validate_pcfg_indicator`)
* spanning     spanning.py:606-666 (`_arcs_to_parent`, `is_projective`, `validate_tree_indicator`)

These are O(size of the indicator) host loops; they never touch the device.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidProblem
from .families import PCFG, CTCDist, LinearChainCRF, MonotoneAlignmentCRF, SemiMarkovCRF, SpanningTreeCRF, TreeCRF

# alignment moves are scored on arrival: DIAG from (i-1, j-1), DOWN from (i-1, j), RIGHT from (i, j-1)
_MOVE_DELTA = ((-1, -1), (-1, 0), (0, -1))
BLANK = 0


def _shape(mask, want, msg):
    if mask.shape != tuple(want):
        raise InvalidProblem(msg)


def chain_tags(d: LinearChainCRF, ind) -> np.ndarray:
    init, trans = ind["init"], ind["transitions"]
    if init.shape != d.init.shape or trans.shape != d.transitions.shape:
        raise InvalidProblem("indicator shape does not match chain potentials")
    if np.count_nonzero(init) != 1:
        raise InvalidProblem("chain indicator must mark exactly one initial tag")
    tags = np.empty(d.n, dtype=np.int64)
    tags[0] = int(np.flatnonzero(init)[0])
    for t in range(d.n - 1):
        hot = np.flatnonzero(trans[t] > 0)
        if hot.size != 1:
            raise InvalidProblem(f"chain indicator must mark one transition at step {t}")
        a, b = divmod(int(hot[0]), d.m)
        if a != tags[t]:
            raise InvalidProblem(f"chain indicator is disconnected at step {t}")
        tags[t + 1] = b
    return tags


def semi_markov_segments(d: SemiMarkovCRF, ind):
    mask = ind["segment_potentials"]
    _shape(mask, d.segment_potentials.shape, "indicator shape does not match segment potentials")
    pos, prev = 0, 0
    segs = []
    # np.argwhere enumerates in lexicographic (start, width-1, prev, label) order
    for t, w, p, lab in np.argwhere(mask > 0):
        if t != pos or p != prev:
            raise InvalidProblem("segments do not tile the sequence consistently")
        segs.append((int(t), int(w) + 1, int(p), int(lab)))
        pos += int(w) + 1
        prev = int(lab)
    if pos != d.n:
        raise InvalidProblem("segments do not cover the full sequence")
    return segs


def alignment_path(d: MonotoneAlignmentCRF, ind):
    mask = ind["move_potentials"]
    _shape(mask, d.move_potentials.shape, "indicator shape does not match move potentials")
    marked = int(np.count_nonzero(mask))
    i, j = d.n, d.m
    steps = 0
    while i != 0 or j != 0:
        hot = np.flatnonzero(mask[i, j] > 0)
        if hot.size != 1:
            raise InvalidProblem(f"path indicator must mark exactly one move into ({i}, {j})")
        di, dj = _MOVE_DELTA[int(hot[0])]
        i, j = i + di, j + dj
        if i < 0 or j < 0:
            raise InvalidProblem("path indicator steps outside the grid")
        steps += 1
    if steps != marked:
        raise InvalidProblem("path indicator marks moves off the path")


def collapse(path, blank: int = BLANK) -> tuple:
    """Merge runs of equal labels, then drop blanks."""
    out = []
    last = None
    for x in path:
        if x != last and x != blank:
            out.append(x)
        last = x
    return tuple(out)


def ctc_path(d: CTCDist, ind):
    mask = ind["frame_potentials"]
    _shape(mask, d.frame_potentials.shape, "indicator shape does not match frame potentials")
    if not np.all(np.count_nonzero(mask, axis=1) == 1):
        raise InvalidProblem("CTC indicator must mark exactly one label per frame")
    path = [int(v) for v in np.argmax(mask, axis=1)]
    if collapse(path) != tuple(d.target):
        raise InvalidProblem("CTC indicator path does not collapse to the target")


def is_binary_bracketing(spans: set, n: int) -> bool:
    """True iff `spans` is exactly the 2n-1 node spans of one binary tree
    over n leaves (constituency.py:143-164).  Iterative: a span is derivable
    iff some split has both halves present and derivable; memoised by span."""
    if len(spans) != 2 * n - 1 or (0, n - 1) not in spans:
        return False
    if any((i, i) not in spans for i in range(n)):
        return False
    ok = {(i, i) for i in range(n)}
    for w in range(1, n):
        for (i, j) in spans:
            if j - i != w:
                continue
            if any((i, k) in ok and (k + 1, j) in ok for k in range(i, j)):
                ok.add((i, j))
    return (0, n - 1) in ok


def tree_spans(d: TreeCRF, ind):
    mask = ind["span_potentials"]
    _shape(mask, d.span_potentials.shape, "indicator shape does not match span potentials")
    per = mask.sum(axis=2)
    if np.any((per != 0) & (per != 1)):
        raise InvalidProblem("each marked span must carry exactly one label")
    spans = {(int(i), int(j)) for i, j in np.argwhere(per > 0)}
    if not is_binary_bracketing(spans, d.n):
        raise InvalidProblem("marked spans do not form a binary bracketing")


def pcfg_spans(d: PCFG, ind):
    mask = ind["sticky"]
    if mask.shape != (d.n, d.n):
        raise InvalidProblem("indicator span mask must have shape [n, n]")
    spans = {(int(i), int(j)) for i, j in np.argwhere(mask > 0)}
    if not is_binary_bracketing(spans, d.n):
        raise InvalidProblem("marked spans do not form a binary bracketing")
    return spans


def _crossing(a, b) -> bool:
    a1, a2 = sorted(a)
    b1, b2 = sorted(b)
    return a1 < b1 < a2 < b2 or b1 < a1 < b2 < a2


def spanning_parent(d: SpanningTreeCRF, ind) -> np.ndarray:
    mask = ind["adjacency"]
    _shape(mask, d.adjacency.shape, "indicator shape does not match adjacency")
    arcs = sorted((int(h), int(c)) for h, c in np.argwhere(mask > 0))
    parent = np.full(d.n + 1, -1, dtype=np.int64)
    for h, c in arcs:
        if parent[c] != -1:
            raise InvalidProblem(f"node {c} has two heads")
        parent[c] = h
    if np.any(parent[1:] < 0):
        raise InvalidProblem("not every node received a head")
    for start in range(1, d.n + 1):
        node, hops = start, 0
        while node != 0:
            node = int(parent[node])
            hops += 1
            if hops > d.n:
                raise InvalidProblem("indicator edges contain a cycle")
    if d.single_root_edge and int(np.sum(parent == 0)) != 1:
        raise InvalidProblem("indicator must use exactly one root edge")
    if d.projective:
        for x in range(len(arcs)):
            for y in range(x + 1, len(arcs)):
                if _crossing(arcs[x], arcs[y]):
                    raise InvalidProblem("indicator has crossing edges but the tree is projective")
    return parent


_BY_TYPE = {
    LinearChainCRF: chain_tags, SemiMarkovCRF: semi_markov_segments, MonotoneAlignmentCRF: alignment_path,
    CTCDist: ctc_path, TreeCRF: tree_spans, PCFG: pcfg_spans, SpanningTreeCRF: spanning_parent,
}


def validate_indicator(dist, indicator) -> dict:
    """dist.py:224-248: float64 copies of the indicator after the 0/1 check
    and the family's structural check."""
    ind = {k: np.asarray(v, dtype=np.float64) for k, v in indicator.items()}
    for key, mask in ind.items():
        if (~((mask == 0.0) | (mask == 1.0))).any():
            raise InvalidProblem(f"indicator {key!r} entries must be 0 or 1")
    fn = _BY_TYPE.get(type(dist))
    if fn is None:
        raise InvalidProblem(f"unknown distribution type {type(dist).__name__}")
    try:
        fn(dist, ind)
    except KeyError as e:  # a missing indicator part
        raise InvalidProblem(f"indicator is missing part {e.args[0]!r}") from None
    return ind
