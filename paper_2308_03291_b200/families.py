"""Distribution classes, name-for-name and check-for-check with the
reference's frozen dataclasses.  They hold float64 NumPy potentials exactly
like the reference (so `potentials()` / indicators / scores are drop-in);
inference goes to the device through `dist.py` -> `kernels.py` -> C-ABI.

Each class also exposes `batch_key()` (the shape signature under which
instances can be stacked into one batched kernel call) and `stack()`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidProblem

NEG_INF = float("-inf")


def as_log_tensor(values, name: str = "tensor") -> np.ndarray:
    """numerics.py:22-29: float64, -inf allowed, NaN and +inf rejected."""
    arr = np.asarray(values, dtype=np.float64)
    if np.isnan(arr).any():
        raise InvalidProblem(f"{name} contains NaN entries")
    if np.isposinf(arr).any():
        raise InvalidProblem(f"{name} contains +inf entries")
    return arr


@dataclass(frozen=True)
class LinearChainCRF:
    """chain.py:32-61: init [m], transitions [n-1, m, m] (step, prev, next)."""

    init: np.ndarray
    transitions: np.ndarray

    family = "linear_chain"

    def __post_init__(self):
        object.__setattr__(self, "init", as_log_tensor(self.init, "init"))
        object.__setattr__(self, "transitions", as_log_tensor(self.transitions, "transitions"))
        if self.init.ndim != 1 or self.init.shape[0] < 1:
            raise InvalidProblem(f"init must be a non-empty vector, got {self.init.shape}")
        m = self.init.shape[0]
        if self.transitions.ndim != 3 or self.transitions.shape[1:] != (m, m):
            raise InvalidProblem(
                f"transitions must have shape [n-1, {m}, {m}], got {self.transitions.shape}")

    @property
    def n(self) -> int:
        return self.transitions.shape[0] + 1

    @property
    def m(self) -> int:
        return self.init.shape[0]

    def potentials(self):
        return {"init": self.init, "transitions": self.transitions}


@dataclass(frozen=True)
class SemiMarkovCRF:
    """chain.py:214-247: segment_potentials [n, s, m, m] (start, width-1,
    prev label, label)."""

    segment_potentials: np.ndarray

    family = "semi_markov"

    def __post_init__(self):
        object.__setattr__(self, "segment_potentials",
                           as_log_tensor(self.segment_potentials, "segment_potentials"))
        p = self.segment_potentials
        if p.ndim != 4 or p.shape[2] != p.shape[3]:
            raise InvalidProblem(f"segment_potentials must have shape [n, s, m, m], got {p.shape}")
        if not (1 <= p.shape[1] <= p.shape[0]):
            raise InvalidProblem("max segment width s must satisfy 1 <= s <= n")

    @property
    def n(self):
        return self.segment_potentials.shape[0]

    @property
    def s(self):
        return self.segment_potentials.shape[1]

    @property
    def m(self):
        return self.segment_potentials.shape[2]

    def potentials(self):
        return {"segment_potentials": self.segment_potentials}


DIAG, DOWN, RIGHT = 0, 1, 2


@dataclass(frozen=True)
class MonotoneAlignmentCRF:
    """alignment.py:30-59: move_potentials [n+1, m+1, 3] (diag, down,
    right), scored on arrival; out-of-grid moves must be -inf."""

    move_potentials: np.ndarray

    family = "monotone_alignment"

    def __post_init__(self):
        object.__setattr__(self, "move_potentials", as_log_tensor(self.move_potentials, "move_potentials"))
        p = self.move_potentials
        if p.ndim != 3 or p.shape[2] != 3 or p.shape[0] < 2 or p.shape[1] < 2:
            raise InvalidProblem(
                f"move_potentials must have shape [n+1, m+1, 3] with n, m >= 1, got {p.shape}")
        if not np.isneginf(p[0, :, DIAG]).all() or not np.isneginf(p[0, :, DOWN]).all():
            raise InvalidProblem("moves into row 0 from outside the grid must be -inf")
        if not np.isneginf(p[:, 0, DIAG]).all() or not np.isneginf(p[:, 0, RIGHT]).all():
            raise InvalidProblem("moves into column 0 from outside the grid must be -inf")

    @property
    def n(self):
        return self.move_potentials.shape[0] - 1

    @property
    def m(self):
        return self.move_potentials.shape[1] - 1

    def potentials(self):
        return {"move_potentials": self.move_potentials}


BLANK = 0


@dataclass(frozen=True)
class CTCDist:
    """alignment.py:198-228: frame_potentials [T, V] (blank = 0), target
    labels in 1..V-1."""

    frame_potentials: np.ndarray
    target: tuple

    family = "ctc"

    def __post_init__(self):
        object.__setattr__(self, "frame_potentials", as_log_tensor(self.frame_potentials, "frame_potentials"))
        object.__setattr__(self, "target", tuple(int(t) for t in self.target))
        p = self.frame_potentials
        if p.ndim != 2 or p.shape[0] < 1 or p.shape[1] < 1:
            raise InvalidProblem(f"frame_potentials must have shape [T, V], got {p.shape}")
        for t in self.target:
            if not (1 <= t < p.shape[1]):
                raise InvalidProblem(f"target labels must lie in 1..{p.shape[1] - 1}, got {t}")

    @property
    def num_frames(self):
        return self.frame_potentials.shape[0]

    @property
    def vocab_size(self):
        return self.frame_potentials.shape[1]

    def potentials(self):
        return {"frame_potentials": self.frame_potentials}


@dataclass(frozen=True)
class OneToOneMatching:
    """alignment.py:373-390 (argmax-only family; out of the GPU path)."""

    scores: np.ndarray

    family = "one_to_one"

    def __post_init__(self):
        object.__setattr__(self, "scores", as_log_tensor(self.scores, "scores"))
        if self.scores.ndim != 2 or self.scores.shape[0] != self.scores.shape[1]:
            raise InvalidProblem(f"scores must be square, got {self.scores.shape}")

    @property
    def n(self):
        return self.scores.shape[0]

    def potentials(self):
        return {"scores": self.scores}


@dataclass(frozen=True)
class TreeCRF:
    """constituency.py:26-49: span_potentials [n, n, m] (i, j, label), i<=j."""

    span_potentials: np.ndarray

    family = "tree_crf"

    def __post_init__(self):
        object.__setattr__(self, "span_potentials", as_log_tensor(self.span_potentials, "span_potentials"))
        p = self.span_potentials
        if p.ndim != 3 or p.shape[0] != p.shape[1] or p.shape[0] < 1 or p.shape[2] < 1:
            raise InvalidProblem(f"span_potentials must have shape [n, n, m], got {p.shape}")

    @property
    def n(self):
        return self.span_potentials.shape[0]

    @property
    def m(self):
        return self.span_potentials.shape[2]

    def potentials(self):
        return {"span_potentials": self.span_potentials}


@dataclass(frozen=True)
class PCFG:
    """constituency.py:184-243: root [NT], binary_rules [NT, S, S] (children
    index NTs then PTs), emissions [n, PT], optional sticky [n, n] in
    {0, -inf}."""

    root: np.ndarray
    binary_rules: np.ndarray
    emissions: np.ndarray
    sticky: np.ndarray | None = None

    family = "pcfg"

    def __post_init__(self):
        object.__setattr__(self, "root", as_log_tensor(self.root, "root"))
        object.__setattr__(self, "binary_rules", as_log_tensor(self.binary_rules, "binary_rules"))
        object.__setattr__(self, "emissions", as_log_tensor(self.emissions, "emissions"))
        nt = self.root.shape[0] if self.root.ndim == 1 else 0
        pt = self.emissions.shape[1] if self.emissions.ndim == 2 else 0
        if nt < 1 or pt < 1:
            raise InvalidProblem("PCFG needs at least one nonterminal and one preterminal")
        s = nt + pt
        if self.binary_rules.shape != (nt, s, s):
            raise InvalidProblem(
                f"binary_rules must have shape [{nt}, {s}, {s}], got {self.binary_rules.shape}")
        if abs(np.exp(self.root).sum() - 1.0) > 1e-6:
            raise InvalidProblem("exp(root) must sum to 1")
        mass = np.exp(self.binary_rules).reshape(nt, -1).sum(axis=1)
        if np.any(np.abs(mass - 1.0) > 1e-6):
            raise InvalidProblem("exp(binary_rules[parent]) must sum to 1 for each parent")
        if self.sticky is None:
            object.__setattr__(self, "sticky", np.zeros((self.n, self.n)))
        else:
            object.__setattr__(self, "sticky", as_log_tensor(self.sticky, "sticky"))
            if self.sticky.shape != (self.n, self.n):
                raise InvalidProblem(f"sticky must have shape [{self.n}, {self.n}], got {self.sticky.shape}")
            if (~(np.isneginf(self.sticky) | (self.sticky == 0.0))).any():
                raise InvalidProblem("sticky entries must be 0 or -inf")

    @property
    def n(self):
        return self.emissions.shape[0]

    @property
    def num_nt(self):
        return self.root.shape[0]

    @property
    def num_pt(self):
        return self.emissions.shape[1]

    def potentials(self):
        return {"root": self.root, "binary_rules": self.binary_rules,
                "emissions": self.emissions, "sticky": self.sticky}


@dataclass(frozen=True)
class SpanningTreeCRF:
    """spanning.py:41-70: adjacency [n+1, n+1] (head, dependent), node 0 is
    the root; diagonal and column 0 must be -inf."""

    adjacency: np.ndarray
    directed: bool = True
    projective: bool = False
    single_root_edge: bool = False

    family = "spanning_tree"

    def __post_init__(self):
        object.__setattr__(self, "adjacency", as_log_tensor(self.adjacency, "adjacency"))
        a = self.adjacency
        if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 2:
            raise InvalidProblem(f"adjacency must be square with >= 2 nodes, got {a.shape}")
        if not np.isneginf(np.diag(a)).all():
            raise InvalidProblem("adjacency diagonal must be -inf")
        if not np.isneginf(a[:, 0]).all():
            raise InvalidProblem("edges into the root (column 0) must be -inf")
        if not self.directed:
            blk = a[1:, 1:]
            if not np.array_equal(blk, blk.T):
                raise InvalidProblem("asymmetric input in undirected mode")

    @property
    def n(self):
        return self.adjacency.shape[0] - 1

    def potentials(self):
        return {"adjacency": self.adjacency}


def undirected_to_directed(d: SpanningTreeCRF) -> SpanningTreeCRF:
    """spanning.py:73-82: orient every undirected tree away from the root;
    the adjacency already stores both orientations."""
    if d.directed:
        raise InvalidProblem("undirected_to_directed requires an undirected instance")
    return SpanningTreeCRF(d.adjacency, directed=True, projective=d.projective,
                           single_root_edge=d.single_root_edge)


FAMILIES = {
    "linear_chain": LinearChainCRF,
    "semi_markov": SemiMarkovCRF,
    "monotone_alignment": MonotoneAlignmentCRF,
    "ctc": CTCDist,
    "one_to_one": OneToOneMatching,
    "tree_crf": TreeCRF,
    "pcfg": PCFG,
    "spanning_tree": SpanningTreeCRF,
}
