"""Seeded synthetic-instance builders shared by the golden-vector generator,
the parity tests and bench.py.

They follow the reference test builders' conventions
(`/root/reference/pkg/tests/helpers.py:12-87`): i.i.d. N(0,1) draws from
`np.random.default_rng(seed)`, structural -inf exactly where the reference
requires it, log-normalised PCFG root/rules.  Every value is rounded to
float32 first and then held as float64, so the CPU reference (float64) and the
GPU path (float32) see bit-identical inputs.
"""

from __future__ import annotations

import numpy as np

NEG_INF = float("-inf")


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def chain(seed, n, m):
    """helpers.py:12-14 -> (init [m], transitions [n-1,m,m])."""
    rng = np.random.default_rng(seed)
    return f32(rng.normal(size=m)), f32(rng.normal(size=(n - 1, m, m)))


def semi_markov(seed, n, s, m):
    """helpers.py:17-19 -> segment_potentials [n,s,m,m]."""
    rng = np.random.default_rng(seed)
    return f32(rng.normal(size=(n, s, m, m)))


def alignment(seed, n, m):
    """helpers.py:22-29 -> move_potentials [n+1,m+1,3] with the boundary
    moves -inf (alignment.py:45-48)."""
    rng = np.random.default_rng(seed)
    mv = f32(rng.normal(size=(n + 1, m + 1, 3)))
    mv[0, :, 0] = NEG_INF
    mv[0, :, 1] = NEG_INF
    mv[:, 0, 0] = NEG_INF
    mv[:, 0, 2] = NEG_INF
    return mv


def zero_alignment(n, m):
    mv = np.zeros((n + 1, m + 1, 3))
    mv[0, :, 0] = NEG_INF
    mv[0, :, 1] = NEG_INF
    mv[:, 0, 0] = NEG_INF
    mv[:, 0, 2] = NEG_INF
    return mv


def ctc(seed, T, V, L):
    """helpers.py:42-45 -> (frame_potentials [T,V], target tuple in 1..V-1)."""
    rng = np.random.default_rng(seed)
    target = tuple(int(x) for x in rng.integers(1, V, size=L))
    return f32(rng.normal(size=(T, V))), target


def tree(seed, n, m):
    """helpers.py:48-50 -> span_potentials [n,n,m]."""
    rng = np.random.default_rng(seed)
    return f32(rng.normal(size=(n, n, m)))


def _log_normalise_f32(x, axis_sizes):
    """Log-normalise rows in float64, round to float32, then renormalise once
    more in float64 and round again so exp-sums stay within 1e-6 of 1 after
    the float32 rounding (constituency.py:208-212)."""
    for _ in range(2):
        flat = x.reshape(axis_sizes[0], -1)
        mx = flat.max(axis=1, keepdims=True)
        z = mx + np.log(np.exp(flat - mx).sum(axis=1, keepdims=True))
        x = f32((flat - z).reshape(x.shape))
    return x


def pcfg(seed, n, nt, pt):
    """helpers.py:53-58 -> (root [NT], rules [NT,S,S], emissions [n,PT])."""
    rng = np.random.default_rng(seed)
    root = rng.normal(size=nt)
    rules = rng.normal(size=(nt, nt + pt, nt + pt))
    emis = rng.normal(size=(n, pt))
    root = _log_normalise_f32(root[None, :], (1,))[0]
    rules = _log_normalise_f32(rules, (nt,))
    return root, rules, f32(emis)


def spanning(seed, n, directed=True):
    """helpers.py:66-78 -> adjacency [n+1,n+1]; column 0 and the diagonal
    -inf; undirected instances symmetric off-root."""
    rng = np.random.default_rng(seed)
    adj = f32(rng.normal(size=(n + 1, n + 1)))
    adj[:, 0] = NEG_INF
    np.fill_diagonal(adj, NEG_INF)
    if not directed:
        up = np.triu(adj[1:, 1:], 1)
        blk = up + up.T
        np.fill_diagonal(blk, NEG_INF)
        adj[1:, 1:] = blk
    return adj


def zero_spanning(n):
    adj = np.zeros((n + 1, n + 1))
    adj[:, 0] = NEG_INF
    np.fill_diagonal(adj, NEG_INF)
    return adj


# -- batched config builders (per-instance seed base + i) ----


def batch_chain(base, B, n, m):
    xs = [chain(base + i, n, m) for i in range(B)]
    return np.stack([x[0] for x in xs]), np.stack([x[1] for x in xs])


def batch_alignment(base, B, n, m):
    return np.stack([alignment(base + i, n, m) for i in range(B)])


def batch_ctc(base, B, T, V, L):
    xs = [ctc(base + i, T, V, L) for i in range(B)]
    return np.stack([x[0] for x in xs]), np.array([x[1] for x in xs], dtype=np.int64)


def batch_tree(base, B, n, m):
    return np.stack([tree(base + i, n, m) for i in range(B)])


def batch_spanning(base, B, n):
    return np.stack([spanning(base + i, n) for i in range(B)])


def batch_pcfg(base, B, n, nt, pt):
    xs = [pcfg(base + i, n, nt, pt) for i in range(B)]
    return tuple(np.stack([x[k] for x in xs]) for k in range(3))


def batch_semi_markov(base, B, n, s, m):
    return np.stack([semi_markov(base + i, n, s, m) for i in range(B)])


# -- derived-op cases (entropy / cross-entropy / KL / log_prob) --------------


def family_inputs(fam, seed, shape):
    """Inputs of one instance of `fam` as the dict of the class's fields."""
    if fam == "chain":
        init, tr = chain(seed, shape["n"], shape["m"])
        return {"init": init, "transitions": tr}
    if fam == "semi_markov":
        return {"segment_potentials": semi_markov(seed, shape["n"], shape["s"], shape["m"])}
    if fam == "alignment":
        return {"move_potentials": alignment(seed, shape["n"], shape["m"])}
    if fam == "ctc":
        fp, tg = ctc(seed, shape["T"], shape["V"], shape["L"])
        return {"frame_potentials": fp, "target": np.array(tg)}
    if fam == "tree":
        return {"span_potentials": tree(seed, shape["n"], shape["m"])}
    if fam == "pcfg":
        r, ru, e = pcfg(seed, shape["n"], shape["nt"], shape["pt"])
        return {"root": r, "binary_rules": ru, "emissions": e}
    if fam == "spanning":
        return {"adjacency": spanning(seed, shape["n"], shape.get("directed", True))}
    raise KeyError(fam)


def make_dist(mod, fam, inp, flags=None):
    """Construct the distribution of `fam` from an inputs dict with the
    classes of `mod` (the reference `structdist` or the GPU package)."""
    flags = flags or {}
    if fam == "chain":
        return mod.LinearChainCRF(inp["init"], inp["transitions"])
    if fam == "semi_markov":
        return mod.SemiMarkovCRF(inp["segment_potentials"])
    if fam == "alignment":
        return mod.MonotoneAlignmentCRF(inp["move_potentials"])
    if fam == "ctc":
        return mod.CTCDist(inp["frame_potentials"], tuple(int(x) for x in inp["target"]))
    if fam == "tree":
        return mod.TreeCRF(inp["span_potentials"])
    if fam == "pcfg":
        return mod.PCFG(inp["root"], inp["binary_rules"], inp["emissions"])
    if fam == "spanning":
        return mod.SpanningTreeCRF(inp["adjacency"], directed=flags.get("directed", True),
                                   projective=flags.get("projective", False),
                                   single_root_edge=flags.get("single", False))
    raise KeyError(fam)
