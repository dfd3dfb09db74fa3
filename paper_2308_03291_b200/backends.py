"""Per-family adapters between the reference-shaped host objects and the
batched device kernels.

A backend stacks B same-shape instances into [B, ...] tensors, moves them to
the device (one H2D copy per tensor), calls `kernels.*` (C-ABI) and brings
back logZ / marginals / compact argmax structures (one D2H copy per output),
then rebuilds the reference's result types (float64 dicts, dense 0/1
indicators).
"""

from __future__ import annotations

import contextlib
import threading

import numpy as np
import torch

from . import kernels as K
from .errors import InvalidProblem, VacuousDistribution
from .families import (
    PCFG,
    CTCDist,
    LinearChainCRF,
    MonotoneAlignmentCRF,
    SemiMarkovCRF,
    SpanningTreeCRF,
    TreeCRF,
)

NEG_INF = float("-inf")


def _device():
    from .dist import device

    return device()


# Exact mode (dist.set_precision("fp64")): log_partition / marginals / derived
# quantities take float64 potentials to the sdb_*_f64 entry points (fp64 in and
# out, like the reference); argmax and sampling keep their fp32-input kernels
# (their arithmetic is fp64 already).
EXACT = False
# per-thread scoped override (dist._run / dist._argmax route a call to the exact kernels
# without touching the process default) and the per-thread magnitude probe
_TL = threading.local()


def exact_now() -> bool:
    return EXACT or getattr(_TL, "exact", False)


@contextlib.contextmanager
def exact_scope():
    prev = getattr(_TL, "exact", False)
    _TL.exact = True
    try:
        yield
    finally:
        _TL.exact = prev


def pot_dtype():
    return torch.float64 if exact_now() else torch.float32


# dist._run's magnitude probe: while armed (per thread), to_dev records each uploaded
# tensor's largest finite |x| as a device scalar (read once, after the call's results are
# back on the host)
def track_magnitude(on: bool):
    _TL.probe = [] if on else None


def tracked_max() -> float:
    pr = getattr(_TL, "probe", None)
    if not pr:
        return 0.0
    return float(torch.stack(pr).max().item())


def to_dev(arrs, dtype=torch.float32):
    """Stack host arrays -> one pinned host tensor -> one async H2D copy."""
    host = torch.from_numpy(np.ascontiguousarray(np.stack(arrs))).to(dtype)
    if host.numel() and torch.cuda.is_available():
        host = host.pin_memory()
    t = host.to(_device(), non_blocking=True)
    pr = getattr(_TL, "probe", None)
    if pr is not None and t.numel() and t.is_floating_point():
        pr.append(torch.where(torch.isfinite(t), t.abs(), torch.zeros((), dtype=t.dtype, device=t.device))
                      .max().to(torch.float64))
    return t


def to_host(t):
    return None if t is None else t.cpu().numpy()


class Result:
    """Host-side outcome of one batched log-partition / marginals call."""

    def __init__(self, logz, status, marg, vacuous_msg, public_keys=None, dev=None):
        self.logz = np.asarray(logz, dtype=np.float64)
        self.status = np.asarray(status)
        self.marg = marg  # list of dict[str, ndarray] or None
        self.msg = vacuous_msg
        self.public_keys = public_keys
        self.dev = dev  # dict[str, device tensor [B, ...]] when run(dev=True): marginals left on the GPU

    def raise_vacuous(self, i):
        st = int(self.status[i])
        if st == K.ST_INVALID:
            raise InvalidProblem("potentials contain NaN or +inf entries")
        if st == K.ST_VACUOUS:
            raise VacuousDistribution(self.msg)

    def public_marg(self, i):
        m = self.marg[i]
        if self.public_keys is None:
            return m
        return {k: m[k] for k in self.public_keys}


class ArgmaxResult:
    def __init__(self, status, build, vacuous_msg, score=None, score_exact=False):
        self.status = np.asarray(status)
        self._build = build
        self.msg = vacuous_msg
        self._score = score
        self._score_exact = score_exact  # the kernel read the float64 potentials themselves

    def raise_vacuous(self, i):
        Result.raise_vacuous(self, i)

    def indicator(self, i):
        return self._build(i)

    def score_of(self, i, dist, ind):
        # exact mode: the indicator's score over the float64 potentials (dist.py:162),
        # not the kernel's sum over their fp32 rounding
        from .dist import _tiny, structure_score

        # tiny instances score over the float64 potentials as in the exact mode
        # (dist.AUTO_EXACT_SIZE)
        if self._score is not None and (self._score_exact or not (exact_now() or _tiny([dist]))):
            return float(self._score[i])
        return structure_score(dist, ind)


class Backend:
    family = None
    vacuous_msg = "no structure has finite score"

    def batch_key(self, d):
        raise NotImplementedError

    def algo(self, d):
        raise NotImplementedError

    def argmax_algo(self, d):
        raise NotImplementedError

    def log_prob(self, d, ind):
        return None

    sample_algo = "forward-filtering-backward-sampling"

    def sample(self, ds, seeds, num):
        """dist.py:179-212 -> (per instance: list of num indicators, algo)."""
        from .errors import UnsupportedInference

        raise UnsupportedInference(f"sampling {type(ds[0]).__name__} is not on the GPU path")

    @staticmethod
    def _noise(seeds, count, num):
        """The reference's Gumbel stream: np.random.default_rng(seed).gumbel
        drawn element by element (numerics.py:167), num samples back to back."""
        g = np.stack([np.random.default_rng(int(s)).gumbel(size=num * count) for s in seeds])
        return torch.as_tensor(g, dtype=torch.float64).cuda()

    def _sample_status(self, st, msg=None):
        st = to_host(st)
        for i in range(len(st)):
            Result([0.0], st[i:i + 1], None, msg or self.vacuous_msg).raise_vacuous(0)


# ---------------------------------------------------------------- chain


class ChainBackend(Backend):
    """chain.py:32-114 on sdb_chain_fb / sdb_chain_viterbi."""

    vacuous_msg = "no tag sequence has finite score"

    def batch_key(self, d):
        return (d.n, d.m)

    def algo(self, d):
        return "forward"

    def argmax_algo(self, d):
        return "viterbi"

    def _stack(self, ds, dtype=torch.float32):
        """Same-length group -> ([B,m], [B,n-1,m,m], None); a ragged group (dist.batch_map
        with per-instance lengths) -> zero-padded layout + lengths [B] for the kernels."""
        ns = [d.n for d in ds]
        if len(set(ns)) == 1:
            return to_dev([d.init for d in ds], dtype), to_dev([d.transitions for d in ds], dtype), None
        n, m = max(ns), ds[0].m
        tr = np.zeros((len(ds), n - 1, m, m))
        for i, d in enumerate(ds):
            tr[i, : d.n - 1] = d.transitions
        lengths = torch.as_tensor(ns, dtype=torch.int32).to(_device())
        return to_dev([d.init for d in ds]), to_dev(list(tr)), lengths

    def run(self, ds, marginals=True, full=False, dev=False):
        init, trans, lengths = self._stack(ds, pot_dtype())
        logz, mi, mt, st = K.chain_fb(init, trans, marginals, lengths)
        marg = None
        if marginals and dev and lengths is None:
            return Result(to_host(logz), to_host(st), None, self.vacuous_msg, dev={"init": mi, "transitions": mt})
        if marginals:
            mi, mt = to_host(mi).astype(np.float64), to_host(mt).astype(np.float64)
            marg = [{"init": mi[i], "transitions": mt[i, : d.n - 1]} for i, d in enumerate(ds)]
        return Result(to_host(logz), to_host(st), marg, self.vacuous_msg)

    def argmax(self, ds):
        init, trans, lengths = self._stack(ds)
        tags, score, st = K.chain_viterbi(init, trans, lengths)
        tags = to_host(tags)

        def build(i):
            d = ds[i]
            ind_i = np.zeros(d.m)
            ind_i[tags[i, 0]] = 1.0
            ind_t = np.zeros_like(d.transitions)
            t = np.arange(d.n - 1)
            ti = tags[i, : d.n]  # (ragged groups: the tags past this instance's length are padding)
            ind_t[t, ti[:-1], ti[1:]] = 1.0
            return {"init": ind_i, "transitions": ind_t}

        return ArgmaxResult(to_host(st), build, self.vacuous_msg)

    def sample(self, ds, seeds, num):
        init, trans, _ = self._stack(ds)
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("chain", dict(n=d0.n, m=d0.m)), num)
        tags, _, st = K.chain_sample(init, trans, noise, num)
        self._sample_status(st)
        tags = to_host(tags)
        out = []
        for i, d in enumerate(ds):
            inds = []
            for r in range(num):
                ind_i = np.zeros(d.m)
                ind_i[tags[i, r, 0]] = 1.0
                ind_t = np.zeros_like(d.transitions)
                t = np.arange(d.n - 1)
                ind_t[t, tags[i, r, :-1], tags[i, r, 1:]] = 1.0
                inds.append({"init": ind_i, "transitions": ind_t})
            out.append(inds)
        return out, self.sample_algo


# ------------------------------------------------------------- alignment


class AlignmentBackend(Backend):
    """alignment.py:62-167 on sdb_nw_fb / sdb_nw_viterbi."""

    vacuous_msg = "no alignment path has finite score"

    def batch_key(self, d):
        return (d.n, d.m)

    def algo(self, d):
        return "needleman-wunsch"

    def argmax_algo(self, d):
        return "max-plus-needleman-wunsch"

    def run(self, ds, marginals=True, full=False, dev=False):
        th = to_dev([d.move_potentials for d in ds], pot_dtype())
        logz, marg, st = K.nw_fb(th, marginals)
        if marginals and dev:
            return Result(to_host(logz), to_host(st), None, self.vacuous_msg, dev={"move_potentials": marg})
        out = None
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"move_potentials": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, self.vacuous_msg)

    def argmax(self, ds):
        th = to_dev([d.move_potentials for d in ds])
        path, score, st = K.nw_viterbi(th)
        path = to_host(path)

        def build(i):
            mask = np.zeros_like(ds[i].move_potentials)
            ii, jj = np.nonzero(path[i] >= 0)
            mask[ii, jj, path[i][ii, jj]] = 1.0
            return {"move_potentials": mask}

        return ArgmaxResult(to_host(st), build, self.vacuous_msg)


    def sample(self, ds, seeds, num):
        th = to_dev([d.move_potentials for d in ds])
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("alignment", dict(n=d0.n, m=d0.m)), num)
        path, _, st = K.nw_sample(th, noise, num)
        self._sample_status(st)
        path = to_host(path)
        out = []
        for i, d in enumerate(ds):
            inds = []
            for r in range(num):
                mask = np.zeros_like(d.move_potentials)
                ii, jj = np.nonzero(path[i, r] >= 0)
                mask[ii, jj, path[i, r][ii, jj]] = 1.0
                inds.append({"move_potentials": mask})
            out.append(inds)
        return out, self.sample_algo


# ------------------------------------------------------------------- CTC


class CTCBackend(Backend):
    """alignment.py:198-336 on sdb_ctc_fb / sdb_ctc_viterbi."""

    vacuous_msg = "no frame path collapses to the target"

    def batch_key(self, d):
        return (d.num_frames, d.vocab_size, len(d.target))

    def algo(self, d):
        return "ctc-forward"

    def argmax_algo(self, d):
        return "max-plus-ctc"

    def _stack(self, ds, dtype=torch.float32):
        tg = to_dev([np.asarray(d.target, dtype=np.int64).reshape(-1) for d in ds], torch.int32)
        return to_dev([d.frame_potentials for d in ds], dtype), tg

    def run(self, ds, marginals=True, full=False, dev=False):
        fp, tg = self._stack(ds, pot_dtype())
        logz, marg, st = K.ctc_fb(fp, tg, marginals)
        if marginals and dev:
            return Result(to_host(logz), to_host(st), None, self.vacuous_msg, dev={"frame_potentials": marg})
        out = None
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"frame_potentials": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, self.vacuous_msg)

    def argmax(self, ds):
        fp, tg = self._stack(ds)
        labels, score, st = K.ctc_viterbi(fp, tg)
        labels = to_host(labels)

        def build(i):
            mask = np.zeros_like(ds[i].frame_potentials)
            mask[np.arange(mask.shape[0]), labels[i]] = 1.0
            return {"frame_potentials": mask}

        return ArgmaxResult(to_host(st), build, self.vacuous_msg)


    def sample(self, ds, seeds, num):
        fp, tg = self._stack(ds)
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("ctc", dict(T=d0.num_frames)), num)
        states, _, st = K.ctc_sample(fp, tg, noise, num)
        self._sample_status(st)
        states = to_host(states)
        out = []
        for i, d in enumerate(ds):
            lab = np.zeros(2 * len(d.target) + 1, dtype=np.int64)
            lab[1::2] = np.asarray(d.target, dtype=np.int64)
            inds = []
            for r in range(num):
                mask = np.zeros_like(d.frame_potentials)
                mask[np.arange(mask.shape[0]), lab[states[i, r]]] = 1.0
                inds.append({"frame_potentials": mask})
            out.append(inds)
        return out, self.sample_algo


# -------------------------------------------------------------- Tree-CRF


class TreeBackend(Backend):
    """constituency.py:26-133 on sdb_tree_fb / sdb_tree_viterbi."""

    vacuous_msg = "no labeled tree has finite score"

    def batch_key(self, d):
        return (d.n, d.m)

    def algo(self, d):
        return "cky-inside"

    def argmax_algo(self, d):
        return "max-plus-cky"

    def run(self, ds, marginals=True, full=False, dev=False):
        th = to_dev([d.span_potentials for d in ds], pot_dtype())
        logz, marg, st = K.tree_fb(th, marginals)
        if marginals and dev:
            return Result(to_host(logz), to_host(st), None, self.vacuous_msg, dev={"span_potentials": marg})
        out = None
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"span_potentials": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, self.vacuous_msg)

    def argmax(self, ds):
        th = to_dev([d.span_potentials for d in ds])
        labels, score, st = K.tree_viterbi(th)
        labels = to_host(labels)

        def build(i):
            mask = np.zeros_like(ds[i].span_potentials)
            ii, jj = np.nonzero(labels[i] >= 0)
            mask[ii, jj, labels[i][ii, jj]] = 1.0
            return {"span_potentials": mask}

        return ArgmaxResult(to_host(st), build, self.vacuous_msg)


    sample_algo = "cky-sampling"

    def sample(self, ds, seeds, num):
        th = to_dev([d.span_potentials for d in ds])
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("tree", dict(n=d0.n, m=d0.m)), num)
        labels, _, st = K.tree_sample(th, noise, num)
        self._sample_status(st)
        labels = to_host(labels)
        out = []
        for i, d in enumerate(ds):
            inds = []
            for r in range(num):
                mask = np.zeros_like(d.span_potentials)
                ii, jj = np.nonzero(labels[i, r] >= 0)
                mask[ii, jj, labels[i, r][ii, jj]] = 1.0
                inds.append({"span_potentials": mask})
            out.append(inds)
        return out, self.sample_algo


# -------------------------------------------------------- spanning trees


class SpanningBackend(Backend):
    """spanning.py:41-402 flag dispatch (span_log_partition / span_marginals
    / span_argmax, spanning.py:673-706): projective -> sdb_eisner /
    sdb_kuhlmann, non-projective -> sdb_mtt.  Undirected instances reuse the
    adjacency as directed (spanning.py:73-82)."""

    def batch_key(self, d):
        return (d.n, d.directed, d.projective, d.single_root_edge)

    @staticmethod
    def _prefix(d):
        return "" if d.directed else "undirected-reduction+"

    def algo(self, d):
        if d.projective:
            name = "eisner-single-root" if d.single_root_edge else "eisner"
        else:
            name = "mtt-single-root" if d.single_root_edge else "mtt-multi-root"
        return self._prefix(d) + name

    def argmax_algo(self, d):
        name = "kuhlmann-arc-hybrid" if d.projective else "chu-liu-edmonds"
        if d.single_root_edge:
            name = "reweighting+" + name
        return self._prefix(d) + name

    def run(self, ds, marginals=True, full=False, dev=False):
        d0 = ds[0]
        adj = to_dev([d.adjacency for d in ds], pot_dtype())
        if d0.projective:
            logz, marg, st = K.eisner(adj, d0.single_root_edge, marginals)
            msg = "no projective tree has finite score"
        else:
            logz, marg, st = K.mtt(adj, d0.single_root_edge, marginals)
            msg = "no spanning tree has finite score"
        out = None
        if marginals and dev:
            return Result(to_host(logz), to_host(st), None, msg, dev={"adjacency": marg})
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"adjacency": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, msg)

    def argmax(self, ds):
        d0 = ds[0]
        adj = to_dev([d.adjacency for d in ds])
        if d0.projective:
            heads, score, st = K.kuhlmann(adj, d0.single_root_edge)
            msg = "no projective tree has finite score"
        else:  # Chu-Liu-Edmonds (spanning.py:410-509)
            heads, st = K.cle(adj, d0.single_root_edge)
            msg = "no arborescence has finite score"
        heads = to_host(heads)

        def build(i):
            n = ds[i].n
            mask = np.zeros((n + 1, n + 1))
            dep = np.arange(1, n + 1)
            mask[heads[i][1:], dep] = 1.0
            return {"adjacency": mask}

        return ArgmaxResult(to_host(st), build, msg)

    def sample(self, ds, seeds, num, algorithm=None):
        """span_sample (spanning.py:709-728): projective -> Eisner decode with
        Gumbel picks; non-projective -> Wilson's loop-erased walks (default) or
        Colbourn's sequential conditioning, both on the GPU."""
        d0 = ds[0]
        if not d0.projective:
            return self._sample_nonprojective(ds, seeds, num, algorithm)
        if algorithm not in (None, "eisner"):
            raise InvalidProblem(f"sampler {algorithm!r} does not apply to projective trees")
        adj = to_dev([d.adjacency for d in ds])
        noise = self._noise(seeds, K.stream_len("eisner", dict(n=d0.n)), num)
        heads, _, st = K.eisner_decode(adj, d0.single_root_edge, noise, num)
        self._sample_status(st, "no projective tree has finite score")
        heads = to_host(heads)
        out = []
        for i, d in enumerate(ds):
            inds = []
            for r in range(num):
                mask = np.zeros((d.n + 1, d.n + 1))
                mask[heads[i, r, 1:], np.arange(1, d.n + 1)] = 1.0
                inds.append({"adjacency": mask})
            out.append(inds)
        return out, self._prefix(d0) + "eisner-sampling"

    def _sample_nonprojective(self, ds, seeds, num, algorithm):
        """span_sample non-projective (spanning.py:719-728) with Wilson's
        loop-erased walks on the GPU (spanning.py:531-558); single-root first
        draws the root's child from the GPU Matrix-Tree marginals
        (spanning.py:517-528); algorithm="colbourn" -> _sample_colbourn."""
        from .errors import SamplerStepLimit

        if algorithm not in (None, "wilson", "colbourn"):
            raise InvalidProblem(f"unknown spanning-tree sampler {algorithm!r}")
        d0 = ds[0]
        single = d0.single_root_edge
        adj = to_dev([d.adjacency for d in ds])
        logz, marg, st = K.mtt(adj, single, single)
        sth, lz = to_host(st), to_host(logz)
        for i in range(len(ds)):
            Result(lz[i:i + 1], sth[i:i + 1], None, "no spanning tree has finite score").raise_vacuous(0)
            if lz[i] == -np.inf:
                raise VacuousDistribution("no spanning tree has finite score")
        streams = [K.GumbelStream(s) for s in seeds]
        mg = to_host(marg).astype(np.float64) if single else None
        if algorithm == "colbourn":
            return self._sample_colbourn(ds, adj, mg, streams, num)
        n = d0.n
        out = [[] for _ in ds]
        for _ in range(num):
            child = None
            work = adj
            if single:
                child = np.empty(len(ds), dtype=np.int64)
                for i in range(len(ds)):
                    w = np.log(np.maximum(mg[i, 0, 1:], 1e-300))
                    g = streams[i].take(n)
                    child[i] = 1 + int(np.argmax(np.where(w > -np.inf, w + g, -np.inf)))
                work = adj.clone()
                keep = work[torch.arange(len(ds)), 0, torch.as_tensor(child)].clone()
                work[:, 0, :] = float("-inf")
                work[torch.arange(len(ds)), 0, torch.as_tensor(child)] = keep
                child = torch.as_tensor(child, dtype=torch.int32).cuda()
            parent, st2 = K.wilson(work, streams, child)
            s2 = to_host(st2)
            if (s2 == 4).any():
                raise SamplerStepLimit("loop-erased walk exceeded its step cap; weights are near-degenerate")
            par = to_host(parent)
            for i, d in enumerate(ds):
                mask = np.zeros((n + 1, n + 1))
                mask[par[i, 1:], np.arange(1, n + 1)] = 1.0
                out[i].append({"adjacency": mask})
        return out, self._prefix(d0) + "wilson"


    # fp32 Matrix-Tree marginals: a column of a healthy conditioned problem sums to 1 within
    # ~1e-6 relative; the reference's 1e-6 test (fp64) would flag round-off here, so the GPU
    # path tests 1e-3 -- still far below what a degenerate (near-singular) column produces
    COLBOURN_COL_TOL = 1e-3

    def _sample_colbourn(self, ds, adj, mg, streams, num):
        """colbourn_sample_arcs (spanning.py:573-603, root child 517-528): for
        each dependent in order, the Matrix-Tree marginals of the partially
        conditioned weights come from ONE batched mtt_kernel launch over all
        instances; the head is a Gumbel-max pick from the instance's own stream
        (numerics.py:162-168, same draws as the reference) and the column is
        conditioned on the device.  An instance whose conditioned marginals
        degenerate finishes with the GPU loop-erased walks on its conditioned
        weights (spanning.py:592-597)."""
        from .errors import SamplerStepLimit

        d0 = ds[0]
        B, n, single = len(ds), d0.n, d0.single_root_edge
        dev = adj.device
        bi = torch.arange(B, device=dev)
        out = [[] for _ in ds]
        fell = np.zeros(B, dtype=bool)
        for _ in range(num):
            work = adj.clone()
            parent = np.full((B, n + 1), -1, dtype=np.int64)
            if single:  # spanning.py:517-528
                child = np.empty(B, dtype=np.int64)
                for i in range(B):
                    w = np.log(np.maximum(mg[i, 0, 1:], 1e-300))
                    child[i] = 1 + int(np.argmax(w + streams[i].take(n)))
                    parent[i, child[i]] = 0
                ct = torch.as_tensor(child, device=dev)
                keep = work[bi, 0, ct].clone()
                work[:, 0, :] = float("-inf")
                work[bi, 0, ct] = keep
            fell = np.zeros(B, dtype=bool)
            for dep in range(1, n + 1):
                todo = [i for i in range(B) if not fell[i] and parent[i, dep] < 0]
                if not todo:
                    continue
                _, marg, st = K.mtt(work, False, True)
                col = to_host(marg[:, :, dep]).astype(np.float64)
                st = to_host(st)
                sel, heads = [], []
                for i in todo:
                    c = col[i]
                    if st[i] != 0 or not np.isfinite(c).all() or abs(c.sum() - 1.0) > self.COLBOURN_COL_TOL:
                        fell[i] = True
                        continue
                    w = np.log(np.maximum(c, 1e-300))
                    h = int(np.argmax(w + streams[i].take(n + 1)))
                    parent[i, dep] = h
                    sel.append(i)
                    heads.append(h)
                if sel:
                    si = torch.as_tensor(sel, device=dev)
                    hi = torch.as_tensor(heads, device=dev)
                    keep = work[si, hi, dep].clone()
                    work[si, :, dep] = float("-inf")
                    work[si, hi, dep] = keep
            if fell.any():  # spanning.py:592-597: walks on the conditioned weights
                idx = np.nonzero(fell)[0]
                par, st2 = K.wilson(work[torch.as_tensor(idx, device=dev)], [streams[i] for i in idx])
                if (to_host(st2) == 4).any():
                    raise SamplerStepLimit("loop-erased walk exceeded its step cap; weights are near-degenerate")
                par = to_host(par)
                for k, i in enumerate(idx):
                    miss = parent[i] < 0
                    miss[0] = False
                    parent[i, miss] = par[k, miss]
            for i in range(B):
                mask = np.zeros((n + 1, n + 1))
                mask[parent[i, 1:], np.arange(1, n + 1)] = 1.0
                out[i].append({"adjacency": mask})
        name = "colbourn+wilson-fallback" if fell[0] else "colbourn"
        return out, self._prefix(d0) + name


# ------------------------------------------------------------------- PCFG




class PCFGBackend(Backend):
    """constituency.py:184-371 on sdb_pcfg_fb.  marginals() returns the
    constituent (span) marginals under the key "sticky" (dist.py:125-127)."""

    vacuous_msg = "the grammar derives no tree for this sentence"

    def batch_key(self, d):
        return (d.n, d.num_nt, d.num_pt)

    def algo(self, d):
        return "pcfg-inside"

    def argmax_algo(self, d):
        return "max-plus-pcfg"

    def _inputs(self, ds, dtype=torch.float32):
        return (to_dev([d.root for d in ds], dtype), to_dev([d.binary_rules for d in ds], dtype),
                to_dev([d.emissions for d in ds], dtype), to_dev([d.sticky for d in ds], dtype))

    def run(self, ds, marginals=True, full=False, dev=False):
        root, rules, emis, sticky = self._inputs(ds, pot_dtype())
        if full:
            # potential_marginals: all four gradients of pcfg_gradients (constituency.py:292-340)
            logz, g, st = K.pcfg_grad(root, rules, emis, sticky)
            if dev:
                return Result(to_host(logz), to_host(st), None, self.vacuous_msg, public_keys=("sticky",), dev=dict(g))
            gh = {k: to_host(v).astype(np.float64) for k, v in g.items()}
            out = [{k: gh[k][i] for k in ("root", "binary_rules", "emissions", "sticky")} for i in range(len(ds))]
            return Result(to_host(logz), to_host(st), out, self.vacuous_msg, public_keys=("sticky",))
        logz, marg, st = K.pcfg_fb(root, rules, emis, sticky, marginals)
        out = None
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"sticky": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, self.vacuous_msg)

    def log_prob(self, d, ind):
        """dist.py:266-271: log-probability of a bracketing = masked inside -
        inside, both in ONE batched kernel call (the mask rides on sticky)."""
        from .validate import pcfg_spans

        spans = pcfg_spans(d, ind)
        span_mask = np.full((d.n, d.n), -np.inf)
        for i, j in spans:
            span_mask[i, j] = 0.0
        root, rules, emis, sticky = self._inputs([d, d], pot_dtype())
        sticky[0] = sticky[0] + torch.as_tensor(span_mask, dtype=sticky.dtype, device=sticky.device)
        logz, _, st = K.pcfg_fb(root, rules, emis, sticky, marginals=False)
        lz, sth = to_host(logz), to_host(st)
        if (sth == K.ST_INVALID).any():
            raise InvalidProblem("potentials contain NaN or +inf entries")
        if lz[0] == -np.inf:
            return -np.inf, "pcfg-masked-inside"
        return float(lz[0] - lz[1]), "pcfg-masked-inside"

    sample_algo = "pcfg-sampling"

    def sample(self, ds, seeds, num):
        root, rules, emis, sticky = self._inputs(ds)
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("pcfg", dict(n=d0.n, NT=d0.num_nt, PT=d0.num_pt)), num)
        mask, _, st = K.pcfg_sample(root, rules, emis, sticky, noise, num)
        self._sample_status(st)
        mh = to_host(mask).astype(np.float64)
        return [[{"sticky": mh[i, r]} for r in range(num)] for i in range(len(ds))], self.sample_algo

    def argmax(self, ds):
        # pcfg_argmax (constituency.py:366-371): fp64 max-plus chart + first-max walk
        root, rules, emis, sticky = self._inputs(ds, pot_dtype())
        mask, score, st = K.pcfg_viterbi(root, rules, emis, sticky)
        mh = to_host(mask).astype(np.float64)

        def build(i):
            return {"sticky": mh[i]}

        # the PCFG argmax score is pcfg_max_score (dist.py:153-154, 164-165)
        return ArgmaxResult(to_host(st), build, self.vacuous_msg, score=to_host(score), score_exact=True)


# ------------------------------------------------------------ semi-Markov


class SemiMarkovBackend(Backend):
    """chain.py:214-327 on sdb_semimarkov_fb / sdb_semimarkov_viterbi."""

    vacuous_msg = "no labeled segmentation has finite score"

    def batch_key(self, d):
        return (d.n, d.s, d.m)

    def algo(self, d):
        return "semi-markov-forward"

    def argmax_algo(self, d):
        return "semi-markov-viterbi"

    def run(self, ds, marginals=True, full=False, dev=False):
        th = to_dev([d.segment_potentials for d in ds], pot_dtype())
        logz, marg, st = K.semimarkov_fb(th, marginals)
        if marginals and dev:
            return Result(to_host(logz), to_host(st), None, self.vacuous_msg, dev={"segment_potentials": marg})
        out = None
        if marginals:
            mg = to_host(marg).astype(np.float64)
            out = [{"segment_potentials": mg[i]} for i in range(len(ds))]
        return Result(to_host(logz), to_host(st), out, self.vacuous_msg)

    def argmax(self, ds):
        th = to_dev([d.segment_potentials for d in ds])
        seg, cnt, score, st = K.semimarkov_viterbi(th)
        seg, cnt = to_host(seg), to_host(cnt)

        def build(i):
            mask = np.zeros_like(ds[i].segment_potentials)
            for s0, w, p, l in seg[i][: cnt[i]]:
                mask[s0, w - 1, p, l] = 1.0
            return {"segment_potentials": mask}

        return ArgmaxResult(to_host(st), build, self.vacuous_msg)

    def sample(self, ds, seeds, num):
        th = to_dev([d.segment_potentials for d in ds])
        d0 = ds[0]
        noise = self._noise(seeds, K.stream_len("semi_markov", dict(n=d0.n, s=d0.s, m=d0.m)), num)
        seg, cnt, _, st = K.semimarkov_sample(th, noise, num)
        self._sample_status(st)
        seg, cnt = to_host(seg), to_host(cnt)
        out = []
        for i, d in enumerate(ds):
            inds = []
            for r in range(num):
                mask = np.zeros_like(d.segment_potentials)
                for s0, w, p, l in seg[i, r][: cnt[i, r]]:
                    mask[s0, w - 1, p, l] = 1.0
                inds.append({"segment_potentials": mask})
            out.append(inds)
        return out, self.sample_algo


_BACKENDS = {
    SemiMarkovCRF: SemiMarkovBackend(),
    PCFG: PCFGBackend(),
    SpanningTreeCRF: SpanningBackend(),
    TreeCRF: TreeBackend(),
    CTCDist: CTCBackend(),
    LinearChainCRF: ChainBackend(),
    MonotoneAlignmentCRF: AlignmentBackend(),
}


def register(cls, backend):
    _BACKENDS[cls] = backend


def for_dist(d):
    return _BACKENDS.get(type(d))
