"""Reference-side binding: route an installed `structdist` (the reference,
0.1.0) onto the sm_100a kernels without changing its code.

The reference's dispatch (`structdist/dist.py:68-163`) reaches every family
through module attributes (`chain.forward_log_partition`,
`spanning.span_marginals`, ...).  `install(structdist)` replaces exactly those
family functions with GPU-backed versions that convert the reference's
frozen dataclass to this package's (same fields, already validated), run the
batched kernels, and return the reference's own result types and exception
classes.  This is the binding INTEGRATION.md describes; the reference's own
test-suite runs through it (tools/refsuite/).

    import structdist
    from paper_2308_03291_b200 import refshim
    undo = refshim.install(structdist)   # ... structdist.marginals(d) now runs on the B200
    undo()                                # restore the reference functions
"""

from __future__ import annotations

import functools

import numpy as np

from . import dist as gd
from . import errors as ge
from . import families as gf

_FIELDS = {
    "LinearChainCRF": ("init", "transitions"),
    "SemiMarkovCRF": ("segment_potentials",),
    "MonotoneAlignmentCRF": ("move_potentials",),
    "TreeCRF": ("span_potentials",),
}


def to_gpu(d):
    """Reference dataclass -> this package's dataclass (same fields)."""
    name = type(d).__name__
    if name in _FIELDS:
        return getattr(gf, name)(*(getattr(d, f) for f in _FIELDS[name]))
    if name == "CTCDist":
        return gf.CTCDist(d.frame_potentials, tuple(d.target))
    if name == "PCFG":
        return gf.PCFG(d.root, d.binary_rules, d.emissions, d.sticky)
    if name == "SpanningTreeCRF":
        return gf.SpanningTreeCRF(d.adjacency, directed=d.directed, projective=d.projective,
                                  single_root_edge=d.single_root_edge)
    raise TypeError(f"no GPU family for {name}")


def _errors_as(sd):
    """Map this package's exceptions onto the reference's classes."""
    table = ((ge.VacuousDistribution, sd.errors.VacuousDistribution),
             (ge.InvalidProblem, sd.errors.InvalidProblem),
             (ge.UnsupportedInference, sd.errors.UnsupportedInference))

    def wrap(fn):
        @functools.wraps(fn)
        def run(*a, **k):
            try:
                return fn(*a, **k)
            except tuple(t[0] for t in table) as e:
                for ours, theirs in table:
                    if isinstance(e, ours):
                        raise theirs(str(e)) from None
                raise
        return run
    return wrap


def _marg(d):
    return {k: np.asarray(v, dtype=np.float64) for k, v in gd.potential_marginals(to_gpu(d)).items()}


def install(sd, exact: bool = False, warm: bool = True):
    """Patch the reference package `sd` (the imported `structdist`); returns an
    undo callable.  exact=True routes log-partition / marginals through the
    float64 entry points (gd.set_precision("fp64")) so results match the
    reference at its own tolerances.  warm=True brings the device up at install
    (dist.warmup), so the first patched call does not pay the CUDA context /
    module initialisation."""
    wrap = _errors_as(sd)
    prev = gd.get_precision()
    if exact:
        gd.set_precision("fp64")
    if warm:
        gd.warmup()  # the device comes up at install, not inside the first patched call
    ch, al, co, sp = sd.chain, sd.alignment, sd.constituency, sd.spanning
    lz = lambda d: float(gd.log_partition(to_gpu(d)))  # noqa: E731
    am = lambda d: gd.argmax(to_gpu(d))  # noqa: E731

    def pcfg_gradients(g):  # constituency.py:292-340 -> (log Z, the four gradients)
        gg = to_gpu(g)
        return float(gd.log_partition(gg)), {k: np.asarray(v) for k, v in gd.potential_marginals(gg).items()}

    def pcfg_max_score(g):  # constituency.py:275-277
        return float(gd.argmax_info(to_gpu(g))[1])

    def span_log_partition(d):  # spanning.py:673-680
        return gd.log_partition_info(to_gpu(d))

    def span_marginals(d):  # spanning.py:683-692
        m, algo = gd.marginals_info(to_gpu(d))
        return np.asarray(m["adjacency"], dtype=np.float64), algo

    def span_argmax(d):  # spanning.py:695-706
        ind, _, algo = gd.argmax_info(to_gpu(d))
        return ind, algo

    patches = {
        ch: {"forward_log_partition": lz, "chain_marginals": _marg, "chain_argmax": am,
             "semi_markov_log_partition": lz, "semi_markov_marginals": _marg, "semi_markov_argmax": am},
        al: {"nw_log_partition": lz, "nw_marginals": _marg, "nw_argmax": am,
             "ctc_log_partition": lz, "ctc_marginals": _marg, "ctc_argmax": am},
        co: {"cky_log_partition": lz, "tree_marginals": _marg, "tree_argmax": am,
             "pcfg_inside": lz, "pcfg_gradients": pcfg_gradients, "pcfg_argmax": am,
             "pcfg_max_score": pcfg_max_score},
        sp: {"span_log_partition": span_log_partition, "span_marginals": span_marginals,
             "span_argmax": span_argmax},
    }
    saved = []
    for mod, fns in patches.items():
        for name, fn in fns.items():
            saved.append((mod, name, getattr(mod, name)))
            setattr(mod, name, wrap(fn))

    def undo():
        for mod, name, fn in saved:
            setattr(mod, name, fn)
        gd.set_precision(prev)
    return undo
