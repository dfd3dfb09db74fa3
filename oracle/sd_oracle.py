"""CPU oracle: a float64 NumPy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
module, and only as the checker (or the timed CPU baseline) -- never as the
product path.  The product path (`paper_2308_03291_b200`) runs the sm_100a
kernels in `_sdb200.so` and raises if that library is missing.

Every function restates one reference algorithm from `structdist` 0.1.0
(`/root/reference/pkg/src/structdist/*.py`, cited as file:line).  Results are
pinned against golden vectors produced by the unmodified reference
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, checked by
`tests/test_oracle_golden.py`).  The restatement is vectorised along
anti-diagonals / span widths / batch axes where the reference loops cell by
cell, so it is also a fair (faster-than-reference) CPU baseline.

Conventions (numerics.py:32-46): log-sum-exp is max-shifted; an all -inf slice
reduces to -inf, never NaN; an empty axis reduces to -inf.
"""

from __future__ import annotations

import math

import numpy as np

NEG_INF = float("-inf")


class Vacuous(Exception):
    """Mirrors errors.VacuousDistribution (errors.py:16)."""


# ---------------------------------------------------------------------------
# numerics (numerics.py:32-60, 128-159)
# ---------------------------------------------------------------------------


def lse(x, axis):
    """numerics.py:32-46: max-shift logsumexp with all -inf -> -inf."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[axis] == 0:
        return np.full(np.delete(np.array(x.shape), axis), NEG_INF)
    mx = np.max(x, axis=axis, keepdims=True)
    safe = np.where(np.isneginf(mx), 0.0, mx)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.log(np.sum(np.exp(x - safe), axis=axis))
    out = s + np.squeeze(safe, axis=axis)
    return np.where(np.isneginf(np.squeeze(mx, axis=axis)), NEG_INF, out)


def lse_all(x) -> float:
    """numerics.py:49-51."""
    return float(lse(np.ravel(np.asarray(x, dtype=np.float64)), 0))


def maxr(x, axis):
    """numerics.py:54-60 (max-plus reduce; empty -> -inf)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[axis] == 0:
        return np.full(np.delete(np.array(x.shape), axis), NEG_INF)
    return np.max(x, axis=axis)


def signed_log_det(mat):
    """numerics.py:128-159: partial-pivot elimination; a pivot with
    |p| <= 1e-12 * (original row max) gives (0, -inf)."""
    a = np.array(mat, dtype=np.float64)
    n = a.shape[0]
    if n == 0:
        return 1, 0.0
    rmag = np.abs(a).max(axis=1)
    sgn, acc = 1, 0.0
    for k in range(n):
        r = k + int(np.argmax(np.abs(a[k:, k])))
        p = a[r, k]
        if abs(p) <= 1e-12 * max(rmag[r], 1e-300):
            return 0, NEG_INF
        if r != k:
            a[[k, r]] = a[[r, k]]
            rmag[[k, r]] = rmag[[r, k]]
            sgn = -sgn
        if p < 0.0:
            sgn = -sgn
        acc += math.log(abs(p))
        if k + 1 < n:
            a[k + 1 :, k:] -= np.outer(a[k + 1 :, k] / p, a[k, k:])
    return sgn, acc


# ---------------------------------------------------------------------------
# linear-chain CRF (chain.py:64-114); batched over a leading axis
# ---------------------------------------------------------------------------


def chain_alpha(init, trans):
    """chain.py:64-70. init [B,m], trans [B,n-1,m,m] -> alpha [B,n,m]."""
    B, m = init.shape
    n = trans.shape[1] + 1
    al = np.empty((B, n, m))
    al[:, 0] = init
    for t in range(n - 1):
        al[:, t + 1] = lse(al[:, t, :, None] + trans[:, t], 1)
    return al


def chain_beta(init, trans):
    """chain.py:73-77."""
    B, m = init.shape
    n = trans.shape[1] + 1
    be = np.zeros((B, n, m))
    for t in range(n - 2, -1, -1):
        be[:, t] = lse(trans[:, t] + be[:, t + 1, None, :], 2)
    return be


def chain_log_partition(init, trans):
    """chain.py:80-81."""
    return lse(chain_alpha(init, trans)[:, -1], 1)


def chain_marginals(init, trans):
    """chain.py:84-95 -> (logZ [B], p_init [B,m], p_trans [B,n-1,m,m]).
    Vacuous instances get logZ=-inf and zero marginals (the API raises)."""
    al = chain_alpha(init, trans)
    be = chain_beta(init, trans)
    z = lse(al[:, -1], 1)
    zz = np.where(np.isneginf(z), 0.0, z)
    with np.errstate(invalid="ignore"):
        pi = np.exp(init + be[:, 0] - zz[:, None])
        pt = np.exp(al[:, :-1, :, None] + trans + be[:, 1:, None, :] - zz[:, None, None, None])
    vac = np.isneginf(z)
    pi[vac] = 0.0
    pt[vac] = 0.0
    return z, pi, pt


def chain_viterbi(init, trans):
    """chain.py:98-114: first-argmax backpointers and final tag.
    Returns (tags [B,n] int, best score [B]); vacuous -> score -inf."""
    B, m = init.shape
    n = trans.shape[1] + 1
    sc = init.copy()
    back = np.zeros((B, n, m), dtype=np.int64)
    for t in range(n - 1):
        cand = sc[:, :, None] + trans[:, t]
        back[:, t + 1] = np.argmax(cand, axis=1)
        sc = np.max(cand, axis=1)
    tags = np.zeros((B, n), dtype=np.int64)
    tags[:, -1] = np.argmax(sc, axis=1)
    for t in range(n - 2, -1, -1):
        tags[:, t] = back[np.arange(B), t + 1, tags[:, t + 1]]
    return tags, np.max(sc, axis=1)


# ---------------------------------------------------------------------------
# semi-Markov CRF (chain.py:250-327); one instance [n,s,m,m]
# ---------------------------------------------------------------------------


def sm_alpha(th):
    """chain.py:250-265: virtual start label 0 at position 0."""
    n, s, m, _ = th.shape
    al = np.full((n + 1, m), NEG_INF)
    al[0, 0] = 0.0
    for t in range(1, n + 1):
        terms = [al[t - w][:, None] + th[t - w, w - 1] for w in range(1, min(s, t) + 1)]
        al[t] = lse(np.concatenate(terms, axis=0), 0)
    return al


def sm_beta(th):
    """chain.py:272-282."""
    n, s, m, _ = th.shape
    be = np.full((n + 1, m), NEG_INF)
    be[n] = 0.0
    for t in range(n - 1, -1, -1):
        terms = [lse(th[t, w - 1] + be[t + w][None, :], 1) for w in range(1, min(s, n - t) + 1)]
        be[t] = lse(np.stack(terms), 0)
    return be


def sm_marginals(th):
    """chain.py:285-298 -> (logZ, marg [n,s,m,m])."""
    n, s, m, _ = th.shape
    al, be = sm_alpha(th), sm_beta(th)
    z = lse_all(al[-1])
    marg = np.zeros_like(th)
    if z == NEG_INF:
        return z, marg
    for t in range(n):
        for w in range(1, min(s, n - t) + 1):
            marg[t, w - 1] = np.exp(al[t][:, None] + th[t, w - 1] + be[t + w][None, :] - z)
    return z, marg


def sm_viterbi(th):
    """chain.py:301-327: per (t,l) the best (w,p) in w-ascending order with a
    strict '>' and first-argmax over p.  Returns (segments, score)."""
    n, s, m, _ = th.shape
    sc = np.full((n + 1, m), NEG_INF)
    sc[0, 0] = 0.0
    back = {}
    for t in range(1, n + 1):
        for l in range(m):
            best, arg = NEG_INF, None
            for w in range(1, min(s, t) + 1):
                cand = sc[t - w] + th[t - w, w - 1, :, l]
                p = int(np.argmax(cand))
                if cand[p] > best:
                    best, arg = cand[p], (w, p)
            sc[t, l] = best
            if arg is not None:
                back[(t, l)] = arg
    best = float(np.max(sc[-1]))
    if best == NEG_INF:
        return [], best
    segs = []
    t, l = n, int(np.argmax(sc[-1]))
    while t > 0:
        w, p = back[(t, l)]
        segs.append((t - w, w, p, l))
        t, l = t - w, p
    return segs[::-1], best


# ---------------------------------------------------------------------------
# monotone alignment (alignment.py:62-167), anti-diagonal vectorised
# moves: 0 DIAG from (i-1,j-1), 1 DOWN from (i-1,j), 2 RIGHT from (i,j-1)
# ---------------------------------------------------------------------------


def _diag_cells(d, n, m):
    i = np.arange(max(0, d - m), min(n, d) + 1)
    return i, d - i


def nw_alpha(th, reduce=lse):
    """alignment.py:62-77 (reduce=lse) and :153-167 (reduce=maxr)."""
    n, m = th.shape[0] - 1, th.shape[1] - 1
    al = np.full((n + 2, m + 2), NEG_INF)  # 1-based pad: al[i+1, j+1]
    al[1, 1] = 0.0
    for d in range(1, n + m + 1):
        i, j = _diag_cells(d, n, m)
        t = np.stack([
            al[i, j] + th[i, j, 0],          # from (i-1, j-1)
            al[i, j + 1] + th[i, j, 1],      # from (i-1, j)
            al[i + 1, j] + th[i, j, 2],      # from (i, j-1)
        ])
        al[i + 1, j + 1] = reduce(t, 0)
    return al[1:, 1:]


def nw_beta(th):
    """alignment.py:84-101."""
    n, m = th.shape[0] - 1, th.shape[1] - 1
    be = np.full((n + 2, m + 2), NEG_INF)
    thp = np.full((n + 2, m + 2, 3), NEG_INF)
    thp[: n + 1, : m + 1] = th
    be[n, m] = 0.0
    for d in range(n + m - 1, -1, -1):
        i, j = _diag_cells(d, n, m)
        t = np.stack([
            thp[i + 1, j + 1, 0] + be[i + 1, j + 1],
            thp[i + 1, j, 1] + be[i + 1, j],
            thp[i, j + 1, 2] + be[i, j + 1],
        ])
        be[i, j] = lse(t, 0)
    return be[: n + 1, : m + 1]


def nw_marginals(th):
    """alignment.py:104-118 -> (logZ, marg [n+1,m+1,3])."""
    n, m = th.shape[0] - 1, th.shape[1] - 1
    al, be = nw_alpha(th), nw_beta(th)
    z = float(al[n, m])
    marg = np.zeros_like(th)
    if z == NEG_INF:
        return z, marg
    alp = np.full((n + 2, m + 2), NEG_INF)
    alp[1:, 1:] = al
    src = np.stack([alp[:-1, :-1], alp[:-1, 1:], alp[1:, :-1]], axis=-1)
    with np.errstate(invalid="ignore"):
        marg = np.exp(src + th + be[:, :, None] - z)
    marg[np.isnan(marg)] = 0.0
    return z, marg


def nw_argmax(th):
    """alignment.py:121-143: max-plus grid, walk back from (n,m), first of
    DIAG, DOWN, RIGHT among in-grid sources.  Returns (mask, score)."""
    n, m = th.shape[0] - 1, th.shape[1] - 1
    al = nw_alpha(th, maxr)
    mask = np.zeros_like(th)
    if al[n, m] == NEG_INF:
        return mask, NEG_INF
    i, j = n, m
    while (i, j) != (0, 0):
        opts = [(k, i + di, j + dj) for k, (di, dj) in enumerate(((-1, -1), (-1, 0), (0, -1)))
                if i + di >= 0 and j + dj >= 0]
        vals = np.array([al[a, b] + th[i, j, k] for k, a, b in opts])
        k, i2, j2 = opts[int(np.argmax(vals))]
        mask[i, j, k] = 1.0
        i, j = i2, j2
    return mask, float(al[n, m])


# ---------------------------------------------------------------------------
# CTC (alignment.py:231-336); batched over instances with equal T, L
# ---------------------------------------------------------------------------


def ctc_labels(targets):
    """alignment.py:231-236: [blank, z1, blank, ..., zL, blank]; [B,2L+1]."""
    targets = np.asarray(targets, dtype=np.int64)
    B, L = targets.shape
    lab = np.zeros((B, 2 * L + 1), dtype=np.int64)
    lab[:, 1::2] = targets
    return lab


def _ctc_skip(lab):
    """alignment.py:239-245: s-2 is a predecessor iff lab[s] != blank and
    lab[s] != lab[s-2]."""
    skip = np.zeros(lab.shape, dtype=bool)
    skip[:, 2:] = (lab[:, 2:] != 0) & (lab[:, 2:] != lab[:, :-2])
    return skip


def ctc_alpha(fp, targets, reduce=lse):
    """alignment.py:248-260. fp [B,T,V] -> alpha [B,T,S]."""
    lab = ctc_labels(targets)
    B, T, _ = fp.shape
    S = lab.shape[1]
    emit = np.take_along_axis(fp, np.broadcast_to(lab[:, None, :], (B, T, S)), axis=2)
    skip = _ctc_skip(lab)
    al = np.full((B, T, S), NEG_INF)
    al[:, 0, 0] = emit[:, 0, 0]
    if S > 1:
        al[:, 0, 1] = emit[:, 0, 1]
    for t in range(1, T):
        p = al[:, t - 1]
        a1 = np.concatenate([np.full((B, 1), NEG_INF), p[:, :-1]], axis=1)
        a2 = np.concatenate([np.full((B, 2), NEG_INF), p[:, :-2]], axis=1)[:, :S]
        a2 = np.where(skip, a2, NEG_INF)
        al[:, t] = reduce(np.stack([p, a1, a2]), 0) + emit[:, t]
    return al, emit, skip


def ctc_log_partition(fp, targets):
    al, _, _ = ctc_alpha(fp, targets)
    S = al.shape[2]
    fin = al[:, -1, -1:] if S == 1 else al[:, -1, S - 2 :]
    return lse(fin, 1)


def ctc_marginals(fp, targets):
    """alignment.py:272-301 -> (logZ [B], marg [B,T,V]); scatter-add of the
    state posteriors by label."""
    al, emit, skip = ctc_alpha(fp, targets)
    lab = ctc_labels(targets)
    B, T, S = al.shape
    V = fp.shape[2]
    be = np.full((B, T, S), NEG_INF)
    be[:, -1, S - 1] = 0.0
    if S > 1:
        be[:, -1, S - 2] = 0.0
    # successor of s: s (stay), s+1 (always), s+2 if skip[s+2]
    skip2 = np.concatenate([skip[:, 2:], np.zeros((B, 2), dtype=bool)], axis=1)[:, :S]
    for t in range(T - 2, -1, -1):
        q = emit[:, t + 1] + be[:, t + 1]
        q1 = np.concatenate([q[:, 1:], np.full((B, 1), NEG_INF)], axis=1)
        q2 = np.concatenate([q[:, 2:], np.full((B, 2), NEG_INF)], axis=1)[:, :S]
        q2 = np.where(skip2, q2, NEG_INF)
        be[:, t] = lse(np.stack([q, q1, q2]), 0)
    fin = al[:, -1, -1:] if S == 1 else al[:, -1, S - 2 :]
    z = lse(fin, 1)
    zz = np.where(np.isneginf(z), 0.0, z)
    with np.errstate(invalid="ignore"):
        post = np.exp(al + be - zz[:, None, None])
    post[np.isnan(post)] = 0.0
    marg = np.zeros((B, T, V))
    for b in range(B):
        for s in range(S):
            marg[b, :, lab[b, s]] += post[b, :, s]
    marg[np.isneginf(z)] = 0.0
    return z, marg


def ctc_argmax(fp, targets):
    """alignment.py:304-336: best expanded-state path; ties go to pred order
    [s, s-1, s-2] and final order [S-1, S-2].  Returns (labels per frame
    [B,T], score [B])."""
    al, emit, skip = ctc_alpha(fp, targets, reduce=maxr)
    lab = ctc_labels(targets)
    B, T, S = al.shape
    out = np.zeros((B, T), dtype=np.int64)
    score = np.full(B, NEG_INF)
    for b in range(B):
        fins = [S - 1] if S == 1 else [S - 1, S - 2]
        vals = [al[b, -1, s] for s in fins]
        if max(vals) == NEG_INF:
            continue
        s = fins[int(np.argmax(vals))]
        score[b] = max(vals)
        states = [s]
        for t in range(T - 1, 0, -1):
            preds = [s] + ([s - 1] if s >= 1 else []) + ([s - 2] if s >= 2 and skip[b, s] else [])
            v = [al[b, t - 1, p] for p in preds]
            s = preds[int(np.argmax(v))]
            states.append(s)
        states.reverse()
        out[b] = lab[b, states]
    return out, score


# ---------------------------------------------------------------------------
# Tree-CRF CKY (constituency.py:52-133); one instance [n,n,m]
# ---------------------------------------------------------------------------


def tree_inside(th, reduce=lse):
    """constituency.py:52-64."""
    n = th.shape[0]
    fold = reduce(th, 2)
    ins = np.full((n, n), NEG_INF)
    idx = np.arange(n)
    ins[idx, idx] = fold[idx, idx]
    for w in range(2, n + 1):
        i = np.arange(0, n - w + 1)
        j = i + w - 1
        k = np.arange(w - 1)
        parts = ins[i[:, None], i[:, None] + k[None, :]] + ins[i[:, None] + k[None, :] + 1, j[:, None]]
        ins[i, j] = fold[i, j] + reduce(parts, 1)
    return fold, ins


def tree_marginals(th):
    """constituency.py:77-110 -> (logZ, marg [n,n,m])."""
    n = th.shape[0]
    fold, ins = tree_inside(th)
    z = float(ins[0, n - 1])
    marg = np.zeros_like(th)
    if z == NEG_INF:
        return z, marg
    out = np.full((n, n), NEG_INF)
    out[0, n - 1] = 0.0
    for w in range(n - 1, 0, -1):
        for i in range(0, n - w + 1):
            j = i + w - 1
            pj = np.arange(j + 1, n)
            pi = np.arange(0, i)
            parts = []
            if pj.size:  # right sibling (j+1, pj)
                parts.append(out[i, pj] + fold[i, pj] + ins[j + 1, pj])
            if pi.size:  # left sibling (pi, i-1)
                parts.append(out[pi, j] + fold[pi, j] + ins[pi, i - 1])
            terms = np.concatenate(parts) if parts else np.zeros(0)
            if terms.size:
                out[i, j] = lse(terms, 0)
    with np.errstate(invalid="ignore"):  # -inf - -inf on spans the mask below drops
        child = ins - fold
    ok = np.isfinite(ins) & np.isfinite(out)
    iu, ju = np.nonzero(np.triu(ok))
    marg[iu, ju] = np.exp(out[iu, ju, None] + child[iu, ju, None] + th[iu, ju] - z)
    return z, marg


def tree_argmax(th):
    """constituency.py:113-133: label = first argmax, split = first argmax of
    inside[i,k] + inside[k+1,j] on the max-plus chart.  Returns (label mask
    [n,n] int with -1 for spans not in the tree, score)."""
    n = th.shape[0]
    _, ins = tree_inside(th, maxr)
    lab = np.full((n, n), -1, dtype=np.int64)
    if ins[0, n - 1] == NEG_INF:
        return lab, NEG_INF
    stack = [(0, n - 1)]
    while stack:
        i, j = stack.pop()
        lab[i, j] = int(np.argmax(th[i, j]))
        if i == j:
            continue
        k = i + int(np.argmax(ins[i, i:j] + ins[i + 1 : j + 1, j]))
        stack += [(i, k), (k + 1, j)]
    return lab, float(ins[0, n - 1])


# ---------------------------------------------------------------------------
# PCFG (constituency.py:246-371); one instance
# ---------------------------------------------------------------------------


def pcfg_inside_chart(root, rules, emis, sticky=None, reduce=lse):
    """constituency.py:246-266. chart [n,n,S]; width-1 cells hold
    preterminals (slots NT..S-1), wider cells nonterminals (0..NT-1)."""
    n, pt = emis.shape
    nt = root.shape[0]
    S = nt + pt
    add = np.zeros((n, n)) if sticky is None else sticky
    ch = np.full((n, n, S), NEG_INF)
    for i in range(n):
        ch[i, i, nt:] = emis[i] + add[i, i]
    for w in range(2, n + 1):
        for i in range(0, n - w + 1):
            j = i + w - 1
            L = ch[i, i:j]
            R = ch[i + 1 : j + 1, j]
            pair = reduce(L[:, :, None] + R[:, None, :], 0)
            inner = reduce(reduce(rules + pair[None], 2), 1)
            ch[i, j, :nt] = inner + add[i, j]
    return ch


def pcfg_log_partition(root, rules, emis, sticky=None):
    """constituency.py:269-272."""
    n = emis.shape[0]
    nt = root.shape[0]
    ch = pcfg_inside_chart(root, rules, emis, sticky)
    return lse_all(root + ch[0, n - 1, :nt])


def pcfg_gradients(root, rules, emis, sticky=None):
    """constituency.py:292-340 -> (logZ, dict root/binary_rules/emissions/
    sticky).  sticky = constituent (span) marginals [n,n]."""
    n, pt = emis.shape
    nt = root.shape[0]
    S = nt + pt
    stk = np.zeros((n, n)) if sticky is None else sticky
    ch = pcfg_inside_chart(root, rules, emis, stk)
    z = lse_all(root + ch[0, n - 1, :nt])
    if z == NEG_INF:
        return z, None
    out = np.full((n, n, S), NEG_INF)
    out[0, n - 1, :nt] = root
    g_rules = np.zeros_like(rules)
    for w in range(n, 1, -1):
        for i in range(0, n - w + 1):
            j = i + w - 1
            o = out[i, j, :nt] + stk[i, j]
            if np.all(np.isneginf(o)):
                continue
            k = np.arange(i, j)
            L = ch[i, k]          # [w-1, S]
            R = ch[k + 1, j]      # [w-1, S]
            orule = o[:, None, None] + rules  # [NT,S,S]
            with np.errstate(invalid="ignore"):
                joint = orule[None] + L[:, None, :, None] + R[:, None, None, :]
                g_rules += np.exp(joint - z).sum(0)
            toL = lse(lse(orule[None] + R[:, None, None, :], 3), 1)  # [w-1,S]
            toR = lse(lse(orule[None] + L[:, None, :, None], 2), 1)
            for a, kk in enumerate(k):
                out[i, kk] = np.logaddexp(out[i, kk], toL[a])
                out[kk + 1, j] = np.logaddexp(out[kk + 1, j], toR[a])
    g_root = np.exp(root + ch[0, n - 1, :nt] - z)
    dout = np.stack([out[i, i, nt:] for i in range(n)])
    dst = np.array([stk[i, i] for i in range(n)])
    g_emis = np.exp(dout + dst[:, None] + emis - z)
    span = np.zeros((n, n))
    for i in range(n):
        for j in range(i, n):
            tot = lse_all(out[i, j] + ch[i, j])
            span[i, j] = np.exp(tot - z) if tot > NEG_INF else 0.0
    return z, {"root": g_root, "binary_rules": g_rules, "emissions": g_emis, "sticky": span}


def pcfg_span_marginals(root, rules, emis, sticky=None):
    """constituency.py:292-340 restricted to what `marginals()` returns for a
    PCFG (dist.py:125-127: the span marginals `sticky` only), in the same log
    semiring as the reference, with the splits of a span batched: the outside
    message of a parent span is folded once through the rules,
    Q[B,C] = lse_A(out[A] + rules[A,B,C]) (constituency.py:321-325 summed in
    the other order -- exact in real arithmetic, float64 here), and each split
    k then costs one [S,S] lse.  Used as the host-CPU baseline for C5b (the
    per-split [NT,S,S] temporaries of pcfg_gradients make it ~20x slower);
    checked against pcfg_gradients in tests/test_oracle_golden.py.
    Returns (logZ, span marginals [n,n])."""
    n, pt = emis.shape
    nt = root.shape[0]
    S = nt + pt
    stk = np.zeros((n, n)) if sticky is None else sticky
    ch = pcfg_inside_chart(root, rules, emis, stk)
    z = lse_all(root + ch[0, n - 1, :nt])
    if z == NEG_INF:
        return z, None
    out = np.full((n, n, S), NEG_INF)
    out[0, n - 1, :nt] = root
    for w in range(n, 1, -1):
        for i in range(0, n - w + 1):
            j = i + w - 1
            o = out[i, j, :nt] + stk[i, j]
            if np.all(np.isneginf(o)):
                continue
            qL = lse(o[:, None, None] + rules, 0)  # [S(B), S(C)]
            L = ch[i, i:j]                          # [w-1, S] left children (i, k)
            R = ch[i + 1 : j + 1, j]                # [w-1, S] right children (k+1, j)
            toL = lse(qL[None, :, :] + R[:, None, :], 2)  # [w-1, B]
            toR = lse(qL[None, :, :] + L[:, :, None], 1)  # [w-1, C]
            out[i, i:j] = np.logaddexp(out[i, i:j], toL)
            out[i + 1 : j + 1, j] = np.logaddexp(out[i + 1 : j + 1, j], toR)
    span = np.zeros((n, n))
    tot = lse(out + ch, 2)
    for i in range(n):
        for j in range(i, n):
            span[i, j] = np.exp(tot[i, j] - z) if tot[i, j] > NEG_INF else 0.0
    return z, span


def pcfg_argmax(root, rules, emis, sticky=None):
    """constituency.py:343-371: max-plus chart then a top-down walk picking
    the first flat argmax of rules[a] + left + right over (k, B, C).
    Returns (span mask [n,n], best derivation score)."""
    n = emis.shape[0]
    nt = root.shape[0]
    ch = pcfg_inside_chart(root, rules, emis, sticky, reduce=maxr)
    top = root + ch[0, n - 1, :nt]
    mask = np.zeros((n, n))
    if np.max(top) == NEG_INF:
        return mask, NEG_INF
    stack = [(0, n - 1, int(np.argmax(top)))]
    while stack:
        i, j, a = stack.pop()
        mask[i, j] = 1.0
        if i == j:
            continue
        L = ch[i, i:j]
        R = ch[i + 1 : j + 1, j]
        joint = rules[a][None, :, :] + L[:, :, None] + R[:, None, :]
        ko, b, c = np.unravel_index(int(np.argmax(joint.ravel())), joint.shape)
        k = i + int(ko)
        stack += [(i, k, int(b)), (k + 1, j, int(c))]
    return mask, float(np.max(top))


# ---------------------------------------------------------------------------
# spanning trees (spanning.py:90-402); one instance [n+1,n+1]
# ---------------------------------------------------------------------------


def _mtt_weights(adj):
    """spanning.py:90-103: per-column max-shifted exp of incoming edges."""
    n = adj.shape[0] - 1
    inc = adj[:, 1:].copy()
    inc[np.arange(1, n + 1), np.arange(n)] = NEG_INF
    sh = inc.max(axis=0)
    if np.isneginf(sh).any():
        return None
    return np.exp(inc - sh[None]), sh


def _mtt_laplacian(W, single_root):
    """spanning.py:106-120."""
    nr = W[1:]
    if single_root:
        L = np.diag(nr.sum(0)) - nr
        L[0] = W[0]
    else:
        L = np.diag(W.sum(0)) - nr
    return L


def mtt_log_partition(adj, single_root=False):
    """spanning.py:123-136."""
    prep = _mtt_weights(adj)
    if prep is None:
        return NEG_INF
    W, sh = prep
    sgn, la = signed_log_det(_mtt_laplacian(W, single_root))
    if sgn <= 0:
        return NEG_INF
    return la + float(sh.sum())


def mtt_marginals(adj, single_root=False):
    """spanning.py:139-175 (vectorised form of the (dep, head) loop)."""
    n = adj.shape[0] - 1
    prep = _mtt_weights(adj)
    if prep is None:
        raise Vacuous("no spanning tree has finite score")
    W, _ = prep
    inv = np.linalg.inv(_mtt_laplacian(W, single_root))
    marg = np.zeros((n + 1, n + 1))
    dg = np.diag(inv)  # inv[d,d]
    if single_root:
        marg[0, 1:] = W[0] * inv[:, 0]
        t = np.where(np.arange(n)[None, :] != 0, dg[None, :], 0.0) \
            - np.where(np.arange(n)[:, None] != 0, inv.T, 0.0)   # [h, d]
    else:
        marg[0, 1:] = W[0] * dg
        t = dg[None, :] - inv.T                                  # [h, d]
    blk = W[1:] * t
    np.fill_diagonal(blk, 0.0)
    marg[1:, 1:] = blk
    return np.clip(marg, 0.0, 1.0)


def eisner_charts(th, reduce=lse):
    """spanning.py:183-207: cr/cl complete, ir/il incomplete (size n+1)."""
    N = th.shape[0]
    cr = np.full((N, N), NEG_INF)
    cl = np.full((N, N), NEG_INF)
    ir = np.full((N, N), NEG_INF)
    il = np.full((N, N), NEG_INF)
    d = np.arange(N)
    cr[d, d] = 0.0
    cl[d, d] = 0.0
    for w in range(1, N):
        i = np.arange(0, N - w)
        j = i + w
        k = np.arange(w)  # offsets 0..w-1
        ii, kk = i[:, None], i[:, None] + k[None, :]
        fold = reduce(cr[ii, kk] + cl[kk + 1, j[:, None]], 1)
        ir[i, j] = th[i, j] + fold
        il[i, j] = th[j, i] + fold
        cr[i, j] = reduce(ir[ii, kk + 1] + cr[kk + 1, j[:, None]], 1)
        cl[i, j] = reduce(cl[ii, kk] + il[kk, j[:, None]], 1)
    return cr, cl, ir, il


def _root_terms(th, cl, cr):
    """spanning.py:210-212."""
    n = th.shape[0] - 1
    c = np.arange(1, n + 1)
    return th[0, c] + cl[1, c] + cr[c, n]


def eisner_log_partition(adj, single_root=False):
    """spanning.py:215-221."""
    n = adj.shape[0] - 1
    cr, cl, _, _ = eisner_charts(adj)
    if single_root:
        return lse_all(_root_terms(adj, cl, cr))
    return float(cr[0, n])


def eisner_marginals(adj, single_root=False):
    """spanning.py:224-280 restated as a log-space outside pass over the four
    charts (the gradient the reference's linear-space adjoint computes).
    Returns (logZ, marg [n+1,n+1]) clipped to [0,1]."""
    N = adj.shape[0]
    n = N - 1
    cr, cl, ir, il = eisner_charts(adj)
    ocr = np.full((N, N), NEG_INF)
    ocl = np.full((N, N), NEG_INF)
    oir = np.full((N, N), NEG_INF)
    oil = np.full((N, N), NEG_INF)
    marg = np.zeros((N, N))
    if single_root:
        terms = _root_terms(adj, cl, cr)
        z = lse_all(terms)
        if z == NEG_INF:
            return z, marg
        c = np.arange(1, n + 1)
        marg[0, c] = np.where(np.isfinite(terms), np.exp(terms - z), 0.0)
        # d terms / d cl[1,c] and d cr[c,n]
        ocl[1, c] = np.logaddexp(ocl[1, c], adj[0, c] + cr[c, n])
        ocr[c, n] = np.logaddexp(ocr[c, n], adj[0, c] + cl[1, c])
    else:
        z = float(cr[0, n])
        if z == NEG_INF:
            return z, marg
        ocr[0, n] = 0.0
    for w in range(N - 1, 0, -1):
        for i in range(0, N - w):
            j = i + w
            # cl[i,j] = lse_k cl[i,k] + il[k,j], k in [i, j)
            if np.isfinite(ocl[i, j]):
                k = np.arange(i, j)
                o = ocl[i, j]
                ocl[i, k] = np.logaddexp(ocl[i, k], o + il[k, j])
                oil[k, j] = np.logaddexp(oil[k, j], o + cl[i, k])
            # cr[i,j] = lse_k ir[i,k] + cr[k,j], k in (i, j]
            if np.isfinite(ocr[i, j]):
                k = np.arange(i + 1, j + 1)
                o = ocr[i, j]
                oir[i, k] = np.logaddexp(oir[i, k], o + cr[k, j])
                ocr[k, j] = np.logaddexp(ocr[k, j], o + ir[i, k])
            # il[i,j] = th[j,i] + fold, ir[i,j] = th[i,j] + fold
            ofold = np.logaddexp(oil[i, j] + adj[j, i], oir[i, j] + adj[i, j])
            if np.isfinite(oil[i, j]) and np.isfinite(il[i, j]):
                marg[j, i] = np.exp(oil[i, j] + il[i, j] - z)
            if np.isfinite(oir[i, j]) and np.isfinite(ir[i, j]):
                marg[i, j] = np.exp(oir[i, j] + ir[i, j] - z)
            if np.isfinite(ofold):
                k = np.arange(i, j)
                ocr[i, k] = np.logaddexp(ocr[i, k], ofold + cl[k + 1, j])
                ocl[k + 1, j] = np.logaddexp(ocl[k + 1, j], ofold + cr[i, k])
    return z, np.clip(marg, 0.0, 1.0)


def reweight_root(adj):
    """spanning.py:339-350."""
    fin = adj[np.isfinite(adj)]
    if fin.size == 0:
        raise Vacuous("no edge has finite score")
    n = adj.shape[0] - 1
    c = n * (float(fin.max()) - float(fin.min())) + 1.0
    out = adj.copy()
    out[0, 1:] = out[0, 1:] - c
    return out


def kuhlmann_heads(adj, single_root=False):
    """spanning.py:353-402: tabulated arc-hybrid argmax.  Candidates are
    scanned k ascending, head i before head j, strict '>' (equivalently the
    first maximum).  Returns heads [n+1] (heads[0] = -1) or None if vacuous."""
    th = reweight_root(adj) if single_root else adj
    n = th.shape[0] - 1
    N = n + 2
    sc = np.full((N, N), NEG_INF)
    sc[: n + 1, 1 : n + 1] = th[:, 1:]
    tab = np.full((N, N), NEG_INF)
    back = {}
    for i in range(N - 1):
        tab[i, i + 1] = 0.0
    for w in range(2, N):
        for i in range(0, N - w):
            j = i + w
            k = np.arange(i + 1, j)
            base = tab[i, k] + tab[k, j]
            cand = np.stack([base + sc[i, k], base + sc[j, k]], axis=1).ravel()
            cand = np.where(np.repeat(np.isneginf(base), 2), NEG_INF, cand)
            a = int(np.argmax(cand))
            tab[i, j] = cand[a]
            if cand[a] > NEG_INF:
                back[(i, j)] = (int(k[a // 2]), i if a % 2 == 0 else j)
    if tab[0, N - 1] == NEG_INF:
        return None
    heads = np.full(n + 1, -1, dtype=np.int64)
    stack = [(0, N - 1)]
    while stack:
        i, j = stack.pop()
        if j == i + 1:
            continue
        k, h = back[(i, j)]
        heads[k] = h
        stack += [(i, k), (k, j)]
    if single_root and int(np.sum(heads[1:] == 0)) != 1:
        return None
    return heads


def heads_score(adj, heads):
    """dist.py:251-260 / numerics.py:171-183 for a spanning-tree indicator."""
    d = np.arange(1, adj.shape[0])
    vals = adj[heads[1:], d]
    if np.isneginf(vals).any():
        return NEG_INF
    return float(np.sum(vals))


# ---------------------------------------------------------------------------
# sampling (dist.py:179-212) -- Gumbel-max picks from ONE seeded stream
# ---------------------------------------------------------------------------


def sample_log_categorical(rng, logits):
    """numerics.py:162-168: argmax(where(w > -inf, w + g, -inf)), g = one
    rng.gumbel draw per logit, first maximum."""
    w = np.ravel(np.asarray(logits, dtype=np.float64))
    if not (w > NEG_INF).any():
        raise ValueError("cannot sample: all categorical weights are -inf")
    g = rng.gumbel(size=w.shape)
    return int(np.argmax(np.where(w > NEG_INF, w + g, NEG_INF)))


def chain_sample(init, trans, rng):
    """chain.py:117-129 (forward filtering, backward sampling) -> tags [n]."""
    al = chain_alpha(init[None], trans[None])[0]
    if lse_all(al[-1]) == NEG_INF:
        raise Vacuous("no tag sequence has finite score")
    n = al.shape[0]
    tags = np.zeros(n, dtype=np.int64)
    tags[-1] = sample_log_categorical(rng, al[-1])
    for t in range(n - 2, -1, -1):
        tags[t] = sample_log_categorical(rng, al[t] + trans[t][:, tags[t + 1]])
    return tags


def nw_walk(th, al, pick):
    """alignment.py:121-136 -> path [n+1,m+1] (incoming move or -1)."""
    n, m = th.shape[0] - 1, th.shape[1] - 1
    path = np.full((n + 1, m + 1), -1, dtype=np.int64)
    src = {0: (-1, -1), 1: (-1, 0), 2: (0, -1)}
    i, j = n, m
    while (i, j) != (0, 0):
        moves = [(k, i + di, j + dj) for k, (di, dj) in src.items() if i + di >= 0 and j + dj >= 0]
        k, si, sj = moves[pick(np.array([al[a, b] + th[i, j, kk] for kk, a, b in moves]))]
        path[i, j] = k
        i, j = si, sj
    return path


def nw_sample(th, rng):
    """alignment.py:146-150."""
    al = nw_alpha(th)
    if al[-1, -1] == NEG_INF:
        raise Vacuous("no alignment path has finite score")
    return nw_walk(th, al, lambda w: sample_log_categorical(rng, w))


def ctc_sample(fp, target, rng):
    """alignment.py:304-318, 339-343 -> expanded-lattice state per frame [T]."""
    al, _, skip = ctc_alpha(fp[None], np.asarray(target)[None])
    al, skip = al[0], skip[0]
    T, S = al.shape
    finals = [S - 1] if S == 1 else [S - 1, S - 2]
    if lse_all(al[-1, finals]) == NEG_INF:
        raise Vacuous("no frame path collapses to the target")
    s = finals[sample_log_categorical(rng, al[-1, finals])]
    states = [s]
    for t in range(T - 1, 0, -1):
        preds = [s] + ([s - 1] if s >= 1 else []) + ([s - 2] if s >= 2 and skip[s] else [])
        s = preds[sample_log_categorical(rng, al[t - 1, preds])]
        states.append(s)
    return np.array(states[::-1])


def tree_walk(th, ins, pick):
    """constituency.py:113-126 (LIFO stack: right child first) -> labels [n,n] (-1 = none)."""
    n = th.shape[0]
    lab = np.full((n, n), -1, dtype=np.int64)
    stack = [(0, n - 1)]
    while stack:
        i, j = stack.pop()
        lab[i, j] = pick(th[i, j])
        if i == j:
            continue
        k = i + pick(ins[i, i:j] + ins[i + 1:j + 1, j])
        stack.append((i, k))
        stack.append((k + 1, j))
    return lab


def tree_sample(th, rng):
    """constituency.py:136-140."""
    _, ins = tree_inside(th)
    if ins[0, -1] == NEG_INF:
        raise Vacuous("no labeled tree has finite score")
    return tree_walk(th, ins, lambda w: sample_log_categorical(rng, w))


def eisner_decode(th, single_root, pick=None):
    """spanning.py:283-320: shared top-down reconstruction (pick=None ->
    max-plus charts + first argmax).  Returns heads [n+1] (heads[0] = -1)."""
    is_max = pick is None
    cr, cl, ir, il = eisner_charts(th, maxr if is_max else lse)
    choose = (lambda w: int(np.argmax(w))) if is_max else pick
    n = th.shape[0] - 1
    heads = np.full(n + 1, -1, dtype=np.int64)
    stack = []
    if single_root:
        terms = _root_terms(th, cl, cr)
        if (np.max(terms) if is_max else lse_all(terms)) == NEG_INF:
            raise Vacuous("no projective tree has finite score")
        c = 1 + choose(terms)
        heads[c] = 0
        stack += [("cl", 1, c), ("cr", c, n)]
    else:
        if cr[0, n] == NEG_INF:
            raise Vacuous("no projective tree has finite score")
        stack.append(("cr", 0, n))
    while stack:
        kind, i, j = stack.pop()
        if i == j:
            continue
        if kind == "cr":
            k = i + 1 + choose(ir[i, i + 1:j + 1] + cr[i + 1:j + 1, j])
            stack += [("ir", i, k), ("cr", k, j)]
        elif kind == "cl":
            k = i + choose(cl[i, i:j] + il[i:j, j])
            stack += [("cl", i, k), ("il", k, j)]
        else:
            if kind == "ir":
                heads[j] = i
            else:
                heads[i] = j
            k = i + choose(cr[i, i:j] + cl[i + 1:j + 1, j])
            stack += [("cr", i, k), ("cl", k + 1, j)]
    return heads


def eisner_sample(th, single_root, rng):
    """spanning.py:328-331."""
    return eisner_decode(th, single_root, lambda w: sample_log_categorical(rng, w))


# ---------------------------------------------------------------------------
# non-projective argmax (spanning.py:410-509)
# ---------------------------------------------------------------------------


def _find_cycle(parent):
    """spanning.py:410-425: first cycle (lowest start) of a dep -> head map."""
    resolved = {0}
    for start in sorted(parent):
        if start in resolved:
            continue
        path, in_path, node = [], {}, start
        while node not in resolved and node not in in_path:
            in_path[node] = len(path)
            path.append(node)
            node = parent[node]
        if node in in_path:
            return path[in_path[node]:]
        resolved.update(path)
    return None


def max_arborescence(w):
    """spanning.py:428-499: greedy best incoming edges + cycle contraction."""
    size = w.shape[0]
    bh = {}
    for dep in range(1, size):
        col = w[:, dep].copy()
        col[dep] = NEG_INF
        h = int(np.argmax(col))
        if col[h] == NEG_INF:
            raise Vacuous("no arborescence has finite score")
        bh[dep] = h
    cyc = _find_cycle(bh)
    if cyc is None:
        return bh
    cset = set(cyc)
    keep = [v for v in range(size) if v not in cset]
    nid = {v: i for i, v in enumerate(keep)}
    cs = len(keep)
    nw = np.full((cs + 1, cs + 1), NEG_INF)
    enter, leave = {}, {}
    for u in keep:
        nu = nid[u]
        for v in keep:
            if u != v:
                nw[nu, nid[v]] = w[u, v]
        best, arg = NEG_INF, None
        for v in cyc:
            if w[u, v] == NEG_INF:
                continue
            a = w[u, v] - w[bh[v], v]
            if a > best:
                best, arg = a, v
        if arg is not None:
            nw[nu, cs] = best
            enter[nu] = arg
        if u == 0:
            continue
        best, arg = NEG_INF, None
        for v in cyc:
            if w[v, u] > best:
                best, arg = w[v, u], v
        if arg is not None:
            nw[cs, nu] = best
            leave[nu] = arg
    sub = max_arborescence(nw)
    parent, entry = {}, None
    for nd, nh in sub.items():
        if nd == cs:
            entry = enter[nh]
            parent[entry] = keep[nh]
        elif nh == cs:
            parent[keep[nd]] = leave[nd]
        else:
            parent[keep[nd]] = keep[nh]
    for v in cyc:
        if v != entry:
            parent[v] = bh[v]
    return parent


def cle_heads(adj, single_root=False):
    """spanning.py:502-509 -> heads [n+1] (heads[0] = -1)."""
    w = reweight_root(adj) if single_root else adj
    p = max_arborescence(np.asarray(w, dtype=np.float64))
    n = adj.shape[0] - 1
    heads = np.full(n + 1, -1, dtype=np.int64)
    for d, h in p.items():
        heads[d] = h
    if single_root and int(np.sum(heads[1:] == 0)) != 1:
        raise Vacuous("no arborescence satisfies the single-root constraint")
    return heads


def wilson_sample(adj, single_root, rng):
    """spanning.py:517-558: (single root: draw the root child from the exact
    marginals first) then loop-erased random walks toward the tree.
    Returns heads [n+1]."""
    n = adj.shape[0] - 1
    parent = np.full(n + 1, -1, dtype=np.int64)
    in_tree = np.zeros(n + 1, dtype=bool)
    in_tree[0] = True
    if single_root:
        marg = mtt_marginals(adj, True)
        child = 1 + sample_log_categorical(rng, np.log(np.maximum(marg[0, 1:], 1e-300)))
        keep = adj[0, child]
        adj = adj.copy()
        adj[0, :] = NEG_INF
        adj[0, child] = keep
        parent[child] = 0
        in_tree[child] = True
    for start in range(1, n + 1):
        u = start
        while not in_tree[u]:
            parent[u] = sample_log_categorical(rng, adj[:, u])
            u = parent[u]
        u = start
        while not in_tree[u]:
            in_tree[u] = True
            u = parent[u]
    return parent


COLBOURN_COL_TOL = 1e-6  # spanning.py:591


def colbourn_sample(adj, single_root, rng):
    """spanning.py:567-603 (+ 517-528): condition one dependent at a time on the
    Matrix-Tree marginals of the partially conditioned weights; when those
    degenerate (vacuous, singular, non-finite, or a column not summing to 1
    within 1e-6) finish with loop-erased walks on the conditioned weights
    (spanning.py:592-597).  Returns (heads [n+1], fell_back)."""
    n = adj.shape[0] - 1
    parent = np.full(n + 1, -1, dtype=np.int64)
    adj = adj.copy()
    if single_root:
        marg = mtt_marginals(adj, True)
        child = 1 + sample_log_categorical(rng, np.log(np.maximum(marg[0, 1:], 1e-300)))
        keep = adj[0, child]
        adj[0, :] = NEG_INF
        adj[0, child] = keep
        parent[child] = 0
    for dep in [x for x in range(1, n + 1) if parent[x] < 0]:
        try:
            col = mtt_marginals(adj, False)[:, dep]
            if not np.isfinite(col).all() or abs(col.sum() - 1.0) > COLBOURN_COL_TOL:
                raise Vacuous("conditioned marginals degenerated")
        except (Vacuous, np.linalg.LinAlgError):
            tail = wilson_sample(adj, False, rng)
            for dd in range(1, n + 1):
                if parent[dd] < 0:
                    parent[dd] = tail[dd]
            return parent, True
        h = sample_log_categorical(rng, np.log(np.maximum(col, 1e-300)))
        parent[dep] = h
        keep = adj[h, dep]
        adj[:, dep] = NEG_INF
        adj[h, dep] = keep
    return parent, False


def sm_sample(th, rng):
    """chain.py:330-344 -> segments [(start, width, prev, label)] in walk order."""
    n, s, m, _ = th.shape
    al = sm_alpha(th)
    if lse_all(al[-1]) == NEG_INF:
        raise Vacuous("no labeled segmentation has finite score")
    segs = []
    t = n
    l = sample_log_categorical(rng, al[-1])
    while t > 0:
        widths = list(range(1, min(s, t) + 1))
        logits = np.stack([al[t - w] + th[t - w, w - 1, :, l] for w in widths])
        flat = sample_log_categorical(rng, logits)
        w = widths[flat // m]
        p = flat % m
        segs.append((t - w, w, p, l))
        t, l = t - w, p
    return segs


def pcfg_sample(root, rules, emis, rng, sticky=None):
    """constituency.py:343-363, 374-378 -> span mask [n,n]."""
    n, nt = emis.shape[0], root.shape[0]
    ch = pcfg_inside_chart(root, rules, emis, sticky)
    if lse_all(root + ch[0, n - 1, :nt]) == NEG_INF:
        raise Vacuous("the grammar derives no tree for this sentence")
    mask = np.zeros((n, n))
    pick = lambda w: sample_log_categorical(rng, w)  # noqa: E731
    stack = [(0, n - 1, pick(root + ch[0, n - 1, :nt]))]
    while stack:
        i, j, a = stack.pop()
        mask[i, j] = 1.0
        if i == j:
            continue
        left = ch[i, i:j]
        right = ch[i + 1:j + 1, j]
        joint = rules[a][None, :, :] + left[:, :, None] + right[:, None, :]
        k_off, b, c = np.unravel_index(pick(joint.ravel()), joint.shape)
        k = i + int(k_off)
        stack.append((i, k, int(b)))
        stack.append((k + 1, j, int(c)))
    return mask
