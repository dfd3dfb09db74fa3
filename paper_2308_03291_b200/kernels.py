"""Batched device entry points: thin wrappers that hand raw device pointers
and the current CUDA stream to the C-ABI (include/sdb200.h).

Inputs are torch CUDA tensors with the reference's axis order plus a leading
batch axis; they are made contiguous fp32 (int32 for integer structures).
Outputs are freshly allocated device tensors; `status` follows SDB_ST_*.
No call here ever computes on the CPU.
"""

from __future__ import annotations

import torch

from . import _lib

ST_OK, ST_VACUOUS, ST_INVALID = 0, 1, 2
# kernel size limits (include/sdb200.h); larger problems raise NativeError(SDB_ERR_UNSUPPORTED)
PCFG_MAX_NT, PCFG_MAX_PT = 32, 32


def _require_cuda(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise _lib.NativeUnavailable(f"{name} must be a CUDA tensor (no CPU fallback)")


def f32(t: torch.Tensor, name: str = "tensor") -> torch.Tensor:
    _require_cuda(t, name)
    return t.to(torch.float32).contiguous()


def f64(t: torch.Tensor, name: str = "tensor") -> torch.Tensor:
    _require_cuda(t, name)
    return t.to(torch.float64).contiguous()


def exact(t) -> bool:
    """float64 potentials select the exact-mode entry points (sdb_*_f64):
    fp64 in, fp64 out, the reference's recurrences in fp64 on the GPU."""
    return isinstance(t, torch.Tensor) and t.dtype == torch.float64


def i32(t: torch.Tensor, name: str = "tensor") -> torch.Tensor:
    _require_cuda(t, name)
    return t.to(torch.int32).contiguous()


def ptr(t):
    if t is None or t.numel() == 0:
        return None
    return t.data_ptr()


def stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ----------------------------------------------------------------- chain


def chain_fb(init, trans, marginals: bool = True, lengths=None):
    """chain.py:64-95 batched: init [B,m], trans [B,n-1,m,m] ->
    (logz [B] f64, marg_init [B,m] | None, marg_trans | None, status [B]).
    `lengths` [B] int32 (optional): ragged batch, instance b uses its first
    lengths[b] positions (sdb_chain_fb_lengths; marginals past them are 0).
    float64 init/trans (no lengths): the exact mode, sdb_chain_fb_f64."""
    lib = _lib.load()
    if exact(init) and lengths is None:
        return _chain_fb_f64(lib, init, trans, marginals)
    init, trans = f32(init, "init"), f32(trans, "transitions")
    B, m = init.shape
    n = trans.shape[1] + 1
    dev = init.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    mi = torch.empty_like(init) if marginals else None
    mt = torch.empty_like(trans) if marginals else None
    wsb = lib.sdb_chain_fb_workspace(B, n, m)
    ws = workspace(wsb, dev)
    if lengths is not None:
        lengths = i32(lengths, "lengths")
        rc = lib.sdb_chain_fb_lengths(ptr(init), ptr(trans), ptr(lengths), B, n, m, ptr(logz), ptr(mi), ptr(mt),
                                      ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
        _lib.check(rc, "sdb_chain_fb_lengths")
        return logz, mi, mt, status
    rc = lib.sdb_chain_fb(ptr(init), ptr(trans), B, n, m, ptr(logz), ptr(mi), ptr(mt), ptr(status),
                          ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_chain_fb")
    return logz, mi, mt, status


def _chain_fb_f64(lib, init, trans, marginals):
    init, trans = f64(init, "init"), f64(trans, "transitions")
    B, m = init.shape
    n = trans.shape[1] + 1
    dev = init.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    mi = torch.empty_like(init) if marginals else None
    mt = torch.empty_like(trans) if marginals else None
    ws = workspace(lib.sdb_chain_fb_f64_workspace(B, n, m), dev)
    rc = lib.sdb_chain_fb_f64(ptr(init), ptr(trans), B, n, m, ptr(logz), ptr(mi), ptr(mt), ptr(status), ptr(ws),
                              ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_chain_fb_f64")
    return logz, mi, mt, status


def chain_ragged_supported(n: int, m: int) -> bool:
    """Shapes the per-instance-length chain kernels serve (else pad on the host)."""
    return m <= 32 and (n - 1 + 7) // 8 <= 24


def chain_viterbi(init, trans, lengths=None, stream=None):
    """chain.py:98-114 batched -> (tags [B,n] int32, score [B] f64, status);
    `lengths` as in chain_fb (tags past an instance's length are 0).  `stream`:
    launch there instead of the current stream (outputs are still allocated on
    the current stream: see _concurrent)."""
    lib = _lib.load()
    init, trans = f32(init, "init"), f32(trans, "transitions")
    B, m = init.shape
    n = trans.shape[1] + 1
    dev = init.device
    tags = torch.empty(B, n, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    if lengths is not None:
        lengths = i32(lengths, "lengths")
        rc = lib.sdb_chain_viterbi_lengths(ptr(init), ptr(trans), ptr(lengths), B, n, m, ptr(tags), ptr(score),
                                           ptr(status), stream.cuda_stream if stream else stream_ptr(dev))
        _lib.check(rc, "sdb_chain_viterbi_lengths")
        return tags, score, status
    ws = workspace(lib.sdb_chain_viterbi_workspace(B, n, m), dev)
    if stream is not None:  # freed when this call returns: keep it out of reuse until the side work ends
        ws.record_stream(stream)
    rc = lib.sdb_chain_viterbi(ptr(init), ptr(trans), B, n, m, ptr(tags), ptr(score), ptr(status),
                               ptr(ws), ws.numel(), stream.cuda_stream if stream else stream_ptr(dev))
    _lib.check(rc, "sdb_chain_viterbi")
    return tags, score, status


_SIDE = {}


def _side_stream(dev) -> torch.cuda.Stream:
    s = _SIDE.get(dev.index)
    if s is None:
        s = _SIDE[dev.index] = torch.cuda.Stream(dev)
    return s


def _concurrent(dev, main, side, side_first: bool = True):
    """Run `side(stream)` on a side stream concurrently with `main()` on the
    current stream (fork/join: two stream waits).  Used where both halves of
    one request are latency-bound launches with fewer CTAs than SMs, so they
    share the GPU instead of queueing.  `side` allocates its outputs on the
    CURRENT stream and only launches on the side stream; the join makes every
    later use or free on the current stream ordered after the side work, so no
    per-tensor record_stream bookkeeping is needed."""
    cur = torch.cuda.current_stream(dev)
    st = _side_stream(dev)
    st.wait_stream(cur)
    if side_first:
        rs = side(st)
        rm = main()
    else:
        rm = main()
        rs = side(st)
    cur.wait_stream(st)
    return rm, rs


def chain_fb_viterbi(init, trans, marginals: bool = True):
    """log_partition + marginals (chain.py:64-95) AND argmax (chain.py:98-114)
    in one call: the forward-backward cluster kernel on the current stream,
    the Viterbi kernel concurrently on a side stream (B CTAs each).
    -> ((logz, marg_init, marg_trans, status), (tags, score, status))."""
    init, trans = f32(init, "init"), f32(trans, "transitions")
    return _concurrent(init.device, lambda: chain_fb(init, trans, marginals),
                       lambda st: chain_viterbi(init, trans, stream=st))


# ------------------------------------------------------------- alignment


def nw_fb(theta, marginals: bool = True):
    """alignment.py:62-118 batched: theta [B,n+1,m+1,3] ->
    (logz [B] f64, marg [B,n+1,m+1,3] | None, status)."""
    lib = _lib.load()
    x64 = exact(theta)
    theta = (f64 if x64 else f32)(theta, "move_potentials")
    B, n1, m1, _ = theta.shape
    n, m = n1 - 1, m1 - 1
    dev = theta.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(theta) if marginals else None
    if x64:
        ws = workspace(lib.sdb_nw_fb_f64_workspace(B, n, m) if marginals else 0, dev)
        rc = lib.sdb_nw_fb_f64(ptr(theta), B, n, m, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                               stream_ptr(dev))
        _lib.check(rc, "sdb_nw_fb_f64")
        return logz, marg, status
    ws = workspace(lib.sdb_nw_fb_workspace(B, n, m) if marginals else 0, dev)
    rc = lib.sdb_nw_fb(ptr(theta), B, n, m, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                       stream_ptr(dev))
    _lib.check(rc, "sdb_nw_fb")
    return logz, marg, status


def nw_viterbi(theta):
    """alignment.py:121-167 batched -> (path [B,n+1,m+1] int8 move or -1,
    score [B] f64, status)."""
    lib = _lib.load()
    theta = f32(theta, "move_potentials")
    B, n1, m1, _ = theta.shape
    n, m = n1 - 1, m1 - 1
    dev = theta.device
    path = torch.empty(B, n1, m1, dtype=torch.int8, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_nw_viterbi_workspace(B, n, m), dev)
    rc = lib.sdb_nw_viterbi(ptr(theta), B, n, m, ptr(path), ptr(score), ptr(status), ptr(ws), ws.numel(),
                            stream_ptr(dev))
    _lib.check(rc, "sdb_nw_viterbi")
    return path, score, status


# ------------------------------------------------------------------- CTC


def ctc_fb(frame_potentials, targets, marginals: bool = True):
    """alignment.py:248-301 batched: frame_potentials [B,T,V], targets
    [B,L] -> (logz [B] f64, marg [B,T,V] | None, status)."""
    lib = _lib.load()
    x64 = exact(frame_potentials)
    fp = (f64 if x64 else f32)(frame_potentials, "frame_potentials")
    tg = i32(targets, "targets")
    B, T, V = fp.shape
    L = tg.shape[1]
    dev = fp.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(fp) if marginals else None
    if x64:
        ws = workspace(lib.sdb_ctc_fb_f64_workspace(B, T, V, L) if marginals else 0, dev)
        rc = lib.sdb_ctc_fb_f64(ptr(fp), ptr(tg), B, T, V, L, ptr(logz), ptr(marg), ptr(status), ptr(ws),
                                ws.numel(), stream_ptr(dev))
        _lib.check(rc, "sdb_ctc_fb_f64")
        return logz, marg, status
    ws = workspace(lib.sdb_ctc_fb_workspace(B, T, V, L) if marginals else 0, dev)
    rc = lib.sdb_ctc_fb(ptr(fp), ptr(tg), B, T, V, L, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                        stream_ptr(dev))
    _lib.check(rc, "sdb_ctc_fb")
    return logz, marg, status


def ctc_viterbi(frame_potentials, targets):
    """alignment.py:304-336 batched -> (labels per frame [B,T] int32, score, status)."""
    lib = _lib.load()
    fp = f32(frame_potentials, "frame_potentials")
    tg = i32(targets, "targets")
    B, T, V = fp.shape
    L = tg.shape[1]
    dev = fp.device
    labels = torch.empty(B, T, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_ctc_viterbi_workspace(B, T, V, L), dev)
    rc = lib.sdb_ctc_viterbi(ptr(fp), ptr(tg), B, T, V, L, ptr(labels), ptr(score), ptr(status), ptr(ws),
                             ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_ctc_viterbi")
    return labels, score, status


# -------------------------------------------------------------- Tree-CRF


def tree_fb(span_potentials, marginals: bool = True):
    """constituency.py:52-110 batched: span_potentials [B,n,n,m] ->
    (logz [B] f64, marg [B,n,n,m] | None, status)."""
    lib = _lib.load()
    x64 = exact(span_potentials)
    th = (f64 if x64 else f32)(span_potentials, "span_potentials")
    B, n, _, m = th.shape
    dev = th.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(th) if marginals else None
    if x64:
        ws = workspace(lib.sdb_tree_fb_f64_workspace(B, n, m), dev)
        rc = lib.sdb_tree_fb_f64(ptr(th), B, n, m, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                                 stream_ptr(dev))
        _lib.check(rc, "sdb_tree_fb_f64")
        return logz, marg, status
    ws = workspace(lib.sdb_tree_fb_workspace(B, n, m), dev)
    rc = lib.sdb_tree_fb(ptr(th), B, n, m, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                         stream_ptr(dev))
    _lib.check(rc, "sdb_tree_fb")
    return logz, marg, status


def tree_viterbi(span_potentials):
    """constituency.py:113-133 batched -> (labels [B,n,n] int32 (-1 = not in
    tree), score [B], status)."""
    lib = _lib.load()
    th = f32(span_potentials, "span_potentials")
    B, n, _, m = th.shape
    dev = th.device
    labels = torch.empty(B, n, n, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    rc = lib.sdb_tree_viterbi(ptr(th), B, n, m, ptr(labels), ptr(score), ptr(status), stream_ptr(dev))
    _lib.check(rc, "sdb_tree_viterbi")
    return labels, score, status


# ------------------------------------------------------------ Matrix-Tree


def mtt(adjacency, single_root: bool = False, marginals: bool = True):
    """spanning.py:90-175 batched: adjacency [B,n+1,n+1] ->
    (logz [B] f64, marg [B,n+1,n+1] | None, status)."""
    lib = _lib.load()
    x64 = exact(adjacency)
    adj = (f64 if x64 else f32)(adjacency, "adjacency")
    B, n1, _ = adj.shape
    dev = adj.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(adj) if marginals else None
    if x64:
        ws = workspace(lib.sdb_mtt_f64_workspace(B, n1 - 1), dev)
        rc = lib.sdb_mtt_f64(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(logz), ptr(marg), ptr(status),
                             ptr(ws), ws.numel(), stream_ptr(dev))
        _lib.check(rc, "sdb_mtt_f64")
        return logz, marg, status
    if n1 - 1 <= 128:
        rc = lib.sdb_mtt(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(logz), ptr(marg), ptr(status),
                         stream_ptr(dev))
        _lib.check(rc, "sdb_mtt")
        return logz, marg, status
    ws = workspace(lib.sdb_mtt_ex_workspace(B, n1 - 1), dev)  # general fp64 path (mtt_gen.cu)
    rc = lib.sdb_mtt_ex(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(logz), ptr(marg), ptr(status), ptr(ws),
                        ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_mtt_ex")
    return logz, marg, status


# ---------------------------------------------------- projective (Eisner)


def eisner(adjacency, single_root: bool = False, marginals: bool = True):
    """spanning.py:183-280 batched: adjacency [B,n+1,n+1] ->
    (logz [B] f64, marg [B,n+1,n+1] | None, status)."""
    lib = _lib.load()
    x64 = exact(adjacency)
    adj = (f64 if x64 else f32)(adjacency, "adjacency")
    B, n1, _ = adj.shape
    dev = adj.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(adj) if marginals else None
    if x64:
        rc = lib.sdb_eisner_f64(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(logz), ptr(marg), ptr(status),
                                stream_ptr(dev))
        _lib.check(rc, "sdb_eisner_f64")
        return logz, marg, status
    rc = lib.sdb_eisner(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(logz), ptr(marg), ptr(status),
                        stream_ptr(dev))
    _lib.check(rc, "sdb_eisner")
    return logz, marg, status


def kuhlmann(adjacency, single_root: bool = False, stream=None):
    """spanning.py:339-402 batched -> (heads [B,n+1] int32, score, status);
    `stream` as in chain_viterbi."""
    lib = _lib.load()
    adj = f32(adjacency, "adjacency")
    B, n1, _ = adj.shape
    dev = adj.device
    heads = torch.empty(B, n1, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    rc = lib.sdb_kuhlmann(ptr(adj), B, n1 - 1, 1 if single_root else 0, ptr(heads), ptr(score), ptr(status),
                          stream.cuda_stream if stream else stream_ptr(dev))
    _lib.check(rc, "sdb_kuhlmann")
    return heads, score, status


def eisner_kuhlmann(adjacency, single_root: bool = False, marginals: bool = True):
    """Projective log_partition + marginals (spanning.py:183-280) AND the
    public projective argmax (Kuhlmann, spanning.py:339-402) in one call: the
    Eisner kernels on the current stream, Kuhlmann concurrently on a side
    stream (the Eisner grid's second wave leaves SMs idle); Eisner is
    launched first so its first wave takes every SM (2.333 vs 2.355 ms per
    C4 step with Kuhlmann first).
    -> ((logz, marg, status), (heads, score, status))."""
    _require_cuda(adjacency, "adjacency")
    adj = adjacency.contiguous() if exact(adjacency) else f32(adjacency, "adjacency")
    return _concurrent(adj.device, lambda: eisner(adj, single_root, marginals),
                       lambda st: kuhlmann(adj, single_root, stream=st), side_first=False)


# ------------------------------------------------------------------- PCFG


def pcfg_fb(root, rules, emissions, sticky=None, marginals: bool = True):
    """constituency.py:246-340 batched: root [B,NT], rules [B,NT,S,S],
    emissions [B,n,PT], sticky [B,n,n] | None -> (logz [B] f64,
    span marginals [B,n,n] | None, status)."""
    lib = _lib.load()
    if exact(rules):
        logz, g, status = _pcfg_f64(lib, root, rules, emissions, sticky, marginals, False)
        return logz, (g["sticky"] if g else None), status
    root = f32(root, "root")
    rules = f32(rules, "binary_rules")
    emis = f32(emissions, "emissions")
    st_in = f32(sticky, "sticky") if sticky is not None else None
    B, NT = root.shape
    n, PT = emis.shape[1], emis.shape[2]
    dev = root.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty(B, n, n, dtype=torch.float32, device=dev) if marginals else None
    ws = workspace(lib.sdb_pcfg_fb_workspace(B, n, NT, PT), dev)
    rc = lib.sdb_pcfg_fb(ptr(root), ptr(rules), ptr(emis), ptr(st_in), B, n, NT, PT, ptr(logz), ptr(marg),
                         ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_pcfg_fb")
    return logz, marg, status


def pcfg_grad(root, rules, emissions, sticky=None):
    """constituency.py:292-340 (pcfg_gradients) batched -> (logz [B] f64,
    {"root" [B,NT], "binary_rules" [B,NT,S,S], "emissions" [B,n,PT],
    "sticky" [B,n,n]} fp32, status)."""
    lib = _lib.load()
    if exact(rules):
        return _pcfg_f64(lib, root, rules, emissions, sticky, True, True)
    root = f32(root, "root")
    rules = f32(rules, "binary_rules")
    emis = f32(emissions, "emissions")
    st_in = f32(sticky, "sticky") if sticky is not None else None
    B, NT = root.shape
    n, PT = emis.shape[1], emis.shape[2]
    dev = root.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    g = {"root": torch.empty_like(root), "binary_rules": torch.empty_like(rules), "emissions": torch.empty_like(emis),
         "sticky": torch.empty(B, n, n, dtype=torch.float32, device=dev)}
    ws = workspace(lib.sdb_pcfg_grad_workspace(B, n, NT, PT), dev)
    rc = lib.sdb_pcfg_grad(ptr(root), ptr(rules), ptr(emis), ptr(st_in), B, n, NT, PT, ptr(logz), ptr(g["sticky"]),
                           ptr(g["root"]), ptr(g["binary_rules"]), ptr(g["emissions"]), ptr(status), ptr(ws),
                           ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_pcfg_grad")
    return logz, g, status


def _pcfg_f64(lib, root, rules, emissions, sticky, marginals, grad):
    root, rules, emis = f64(root, "root"), f64(rules, "binary_rules"), f64(emissions, "emissions")
    st_in = f64(sticky, "sticky") if sticky is not None else None
    B, NT = root.shape
    n, PT = emis.shape[1], emis.shape[2]
    dev = root.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    g = None
    if marginals:
        g = {"sticky": torch.empty(B, n, n, dtype=torch.float64, device=dev)}
        if grad:
            g.update(root=torch.empty_like(root), binary_rules=torch.empty_like(rules), emissions=torch.empty_like(emis))
    ws = workspace(lib.sdb_pcfg_f64_workspace(B, n, NT, PT, 1 if grad else 0), dev)
    rc = lib.sdb_pcfg_f64(ptr(root), ptr(rules), ptr(emis), ptr(st_in), B, n, NT, PT, ptr(logz),
                          ptr(g["sticky"]) if g else None, ptr(g["root"]) if grad else None,
                          ptr(g["binary_rules"]) if grad else None, ptr(g["emissions"]) if grad else None,
                          ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_pcfg_f64")
    return logz, g, status


def pcfg_viterbi(root, rules, emissions, sticky=None):
    """constituency.py:275-277, 343-371 batched -> (span_mask [B,n,n] int8,
    score [B] f64 = pcfg_max_score, status); float64 inputs: sdb_pcfg_viterbi_f64."""
    lib = _lib.load()
    x64 = exact(rules)
    cv = f64 if x64 else f32
    root = cv(root, "root")
    rules = cv(rules, "binary_rules")
    emis = cv(emissions, "emissions")
    st_in = cv(sticky, "sticky") if sticky is not None else None
    B, NT = root.shape
    n, PT = emis.shape[1], emis.shape[2]
    dev = root.device
    mask = torch.empty(B, n, n, dtype=torch.int8, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_pcfg_viterbi_workspace(B, n, NT, PT), dev)
    fn = lib.sdb_pcfg_viterbi_f64 if x64 else lib.sdb_pcfg_viterbi
    rc = fn(ptr(root), ptr(rules), ptr(emis), ptr(st_in), B, n, NT, PT, ptr(mask), ptr(score), ptr(status), ptr(ws),
            ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_pcfg_viterbi_f64" if x64 else "sdb_pcfg_viterbi")
    return mask, score, status


# ------------------------------------------------------------ semi-Markov


def semimarkov_fb(segment_potentials, marginals: bool = True):
    """chain.py:250-298 batched: [B,n,s,m,m] -> (logz, marg | None, status)."""
    lib = _lib.load()
    x64 = exact(segment_potentials)
    th = (f64 if x64 else f32)(segment_potentials, "segment_potentials")
    B, n, s, m, _ = th.shape
    dev = th.device
    logz = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    marg = torch.empty_like(th) if marginals else None
    if x64:
        ws = workspace(lib.sdb_semimarkov_fb_f64_workspace(B, n, s, m), dev)
        rc = lib.sdb_semimarkov_fb_f64(ptr(th), B, n, s, m, ptr(logz), ptr(marg), ptr(status), ptr(ws), ws.numel(),
                                       stream_ptr(dev))
        _lib.check(rc, "sdb_semimarkov_fb_f64")
        return logz, marg, status
    rc = lib.sdb_semimarkov_fb(ptr(th), B, n, s, m, ptr(logz), ptr(marg), ptr(status), stream_ptr(dev))
    _lib.check(rc, "sdb_semimarkov_fb")
    return logz, marg, status


def semimarkov_viterbi(segment_potentials):
    """chain.py:301-327 batched -> (segments [B,n,4] int32, num_segments [B],
    score [B], status)."""
    lib = _lib.load()
    th = f32(segment_potentials, "segment_potentials")
    B, n, s, m, _ = th.shape
    dev = th.device
    seg = torch.zeros(B, n, 4, dtype=torch.int32, device=dev)
    cnt = torch.empty(B, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_semimarkov_viterbi_workspace(B, n, s, m), dev)
    rc = lib.sdb_semimarkov_viterbi(ptr(th), B, n, s, m, ptr(seg), ptr(cnt), ptr(score), ptr(status), ptr(ws),
                                    ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_semimarkov_viterbi")
    return seg, cnt, score, status


# -------------------------------------------------------------- sampling


def stream_len(family: str, shape: dict) -> int:
    """Gumbel draws one sample can consume (the C-ABI's per-family bound)."""
    if family == "chain":
        return shape["n"] * shape["m"]
    if family == "alignment":
        return 3 * (shape["n"] + shape["m"])
    if family == "ctc":
        return 2 + 3 * (shape["T"] - 1)
    if family == "tree":
        return (2 * shape["n"] - 1) * shape["m"] + shape["n"] ** 2
    if family == "eisner":
        return shape["n"] + 4 * (shape["n"] + 1) ** 2
    if family == "semi_markov":
        return shape["n"] * shape["s"] * shape["m"] + shape["m"]
    if family == "pcfg":
        S = shape["NT"] + shape["PT"]
        return shape["NT"] + S * S * (shape["n"] * (shape["n"] - 1) // 2)
    raise ValueError(family)


def chain_sample(init, trans, noise, num: int):
    """chain.py:117-129 batched: noise [B, >= num*n*m] fp64 Gumbel stream ->
    (tags [B,num,n] int32, used [B], status)."""
    lib = _lib.load()
    init, trans, noise = f32(init, "init"), f32(trans, "transitions"), f64(noise, "noise")
    B, m = init.shape
    n = trans.shape[1] + 1
    dev = init.device
    tags = torch.empty(B, num, n, dtype=torch.int32, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_chain_sample_workspace(B, n, m), dev)
    rc = lib.sdb_chain_sample(ptr(init), ptr(trans), B, n, m, ptr(noise), noise.shape[1], num, ptr(tags), ptr(used),
                              ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_chain_sample")
    return tags, used, status


def nw_sample(theta, noise, num: int):
    """alignment.py:121-150 batched -> (path [B,num,n+1,m+1] int8, used, status)."""
    lib = _lib.load()
    theta, noise = f32(theta, "move_potentials"), f64(noise, "noise")
    B, n1, m1, _ = theta.shape
    dev = theta.device
    path = torch.empty(B, num, n1, m1, dtype=torch.int8, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_nw_sample_workspace(B, n1 - 1, m1 - 1), dev)
    rc = lib.sdb_nw_sample(ptr(theta), B, n1 - 1, m1 - 1, ptr(noise), noise.shape[1], num, ptr(path), ptr(used),
                           ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_nw_sample")
    return path, used, status


def ctc_sample(frame_potentials, targets, noise, num: int):
    """alignment.py:304-343 batched -> (lattice state per frame [B,num,T], used, status)."""
    lib = _lib.load()
    fp, tg, noise = f32(frame_potentials, "frame_potentials"), i32(targets, "targets"), f64(noise, "noise")
    B, T, V = fp.shape
    L = tg.shape[1]
    dev = fp.device
    states = torch.empty(B, num, T, dtype=torch.int32, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_ctc_sample_workspace(B, T, V, L), dev)
    rc = lib.sdb_ctc_sample(ptr(fp), ptr(tg), B, T, V, L, ptr(noise), noise.shape[1], num, ptr(states), ptr(used),
                            ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_ctc_sample")
    return states, used, status


def tree_sample(span_potentials, noise, num: int):
    """constituency.py:113-140 batched -> (labels [B,num,n,n] (-1 = none), used, status)."""
    lib = _lib.load()
    th, noise = f32(span_potentials, "span_potentials"), f64(noise, "noise")
    B, n, _, m = th.shape
    dev = th.device
    labels = torch.empty(B, num, n, n, dtype=torch.int32, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_tree_sample_workspace(B, n, m), dev)
    rc = lib.sdb_tree_sample(ptr(th), B, n, m, ptr(noise), noise.shape[1], num, ptr(labels), ptr(used), ptr(status),
                             ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_tree_sample")
    return labels, used, status


def eisner_decode(adjacency, single_root: bool = False, noise=None, num: int = 1):
    """spanning.py:283-331 batched: noise None -> eisner_max_arcs (max-plus
    decode), else eisner_sample_arcs -> (heads [B,num,n+1], used, status)."""
    lib = _lib.load()
    adj = f32(adjacency, "adjacency")
    B, N, _ = adj.shape
    dev = adj.device
    noise = f64(noise, "noise") if noise is not None else None
    heads = torch.empty(B, num, N, dtype=torch.int32, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_eisner_decode_workspace(B, N - 1), dev)
    rc = lib.sdb_eisner_decode(ptr(adj), B, N - 1, int(single_root), ptr(noise),
                               noise.shape[1] if noise is not None else 0, num, ptr(heads), ptr(used), ptr(status),
                               ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_eisner_decode")
    return heads, used, status


def cle(adjacency, single_root: bool = False):
    """spanning.py:410-509 batched (Chu-Liu-Edmonds) -> (heads [B,n+1] int32, status)."""
    lib = _lib.load()
    adj = f32(adjacency, "adjacency")
    B, N, _ = adj.shape
    dev = adj.device
    heads = torch.empty(B, N, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_cle_workspace(B, N - 1), dev)
    rc = lib.sdb_cle(ptr(adj), B, N - 1, int(single_root), ptr(heads), ptr(status), ptr(ws), ws.numel(),
                     stream_ptr(dev))
    _lib.check(rc, "sdb_cle")
    return heads, status


class GumbelStream:
    """One instance's Gumbel stream np.random.default_rng(seed).gumbel,
    consumed in order; draws fetched ahead are kept for the next consumer
    (so consecutive samples see exactly the reference's stream)."""

    def __init__(self, seed):
        import numpy as np

        self._np = np
        self.rng = np.random.default_rng(int(seed))
        self.buf = np.empty(0)

    def peek(self, k: int):
        if self.buf.size < k:
            self.buf = self._np.concatenate([self.buf, self.rng.gumbel(size=k - self.buf.size)])
        return self.buf[:k]

    def take(self, k: int):
        out = self.peek(k).copy()
        self.buf = self.buf[k:]
        return out


WILSON_STEP_CAP = 10 ** 7  # spanning.py:38


def wilson(adjacency, streams, root_child=None, chunk_steps: int = 0):
    """spanning.py:531-558 batched: loop-erased walks on the GPU, fed chunk by
    chunk from each instance's GumbelStream -> (parent [B,n+1] int32, status)."""
    import numpy as np

    lib = _lib.load()
    adj = f32(adjacency, "adjacency")
    B, N, _ = adj.shape
    n = N - 1
    dev = adj.device
    parent = torch.empty(B, N, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    used = torch.zeros(B, dtype=torch.int64, device=dev)
    ws = workspace(lib.sdb_wilson_workspace(B, n), dev)
    ch = i32(root_child, "root_child") if root_child is not None else None
    _lib.check(lib.sdb_wilson_begin(B, n, ptr(ch), ptr(parent), ptr(status), ptr(ws), ws.numel(), stream_ptr(dev)),
               "sdb_wilson_begin")
    cap = N * (chunk_steps or 4 * N)
    prev = np.zeros(B, dtype=np.int64)
    while True:
        st = status.cpu().numpy()
        live = st == 3
        if not live.any():
            break
        noise = np.zeros((B, cap))
        for b in np.nonzero(live)[0]:
            noise[b] = streams[b].peek(cap)
        noise_d = torch.as_tensor(noise, device=dev)
        rc = lib.sdb_wilson_step(ptr(adj), B, n, ptr(noise_d), cap, WILSON_STEP_CAP,
                                 ptr(parent), ptr(used), ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
        _lib.check(rc, "sdb_wilson_step")
        u = used.cpu().numpy()
        for b in np.nonzero(live)[0]:
            streams[b].take(int(u[b] - prev[b]))
        prev = u
    return parent, status


def semimarkov_sample(segment_potentials, noise, num: int):
    """chain.py:330-344 batched -> (segments [B,num,n,4], nseg [B,num], used, status)."""
    lib = _lib.load()
    th, noise = f32(segment_potentials, "segment_potentials"), f64(noise, "noise")
    B, n, s, m, _ = th.shape
    dev = th.device
    seg = torch.empty(B, num, n, 4, dtype=torch.int32, device=dev)
    nseg = torch.empty(B, num, dtype=torch.int32, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_semimarkov_sample_workspace(B, n, s, m), dev)
    rc = lib.sdb_semimarkov_sample(ptr(th), B, n, s, m, ptr(noise), noise.shape[1], num, ptr(seg), ptr(nseg),
                                   ptr(used), ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_semimarkov_sample")
    return seg, nseg, used, status


def pcfg_sample(root, rules, emissions, sticky, noise, num: int):
    """constituency.py:374-378 batched -> (span_mask [B,num,n,n] int8, used, status)."""
    lib = _lib.load()
    root = f32(root, "root")
    rules = f32(rules, "binary_rules")
    emis = f32(emissions, "emissions")
    st_in = f32(sticky, "sticky") if sticky is not None else None
    noise = f64(noise, "noise")
    B, NT = root.shape
    n, PT = emis.shape[1], emis.shape[2]
    dev = root.device
    mask = torch.empty(B, num, n, n, dtype=torch.int8, device=dev)
    used = torch.empty(B, dtype=torch.int32, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(lib.sdb_pcfg_viterbi_workspace(B, n, NT, PT), dev)
    rc = lib.sdb_pcfg_sample(ptr(root), ptr(rules), ptr(emis), ptr(st_in), B, n, NT, PT, ptr(noise), noise.shape[1],
                             num, ptr(mask), ptr(used), ptr(status), ptr(ws), ws.numel(), stream_ptr(dev))
    _lib.check(rc, "sdb_pcfg_sample")
    return mask, used, status


# ------------------------------------------------------ derived quantities


def expected_score(pairs, B: int, device):
    """sum_e p(e) theta(e) per instance over (marginals, potentials) device
    tensor pairs with a leading batch axis (dist.py:306-347 via masked_dot,
    numerics.py:171-183) -> (score [B] f64, neginf [B] i32: a marked part
    is -inf).  Only B doubles leave the device."""
    lib = _lib.load()
    out = torch.zeros(B, dtype=torch.float64, device=device)
    flag = torch.zeros(B, dtype=torch.int32, device=device)
    keep = []
    for marg, theta in pairs:
        x64 = exact(marg) or exact(theta)
        cv = f64 if x64 else f32
        marg, theta = cv(marg, "marginals"), cv(theta, "potentials")
        if marg.shape != theta.shape:
            raise ValueError(f"marginals {tuple(marg.shape)} vs potentials {tuple(theta.shape)}")
        keep += [marg, theta]
        fn = lib.sdb_masked_dot_f64 if x64 else lib.sdb_masked_dot
        rc = fn(ptr(marg), ptr(theta), B, marg.numel() // max(B, 1), ptr(out), ptr(flag), stream_ptr(device))
        _lib.check(rc, "sdb_masked_dot_f64" if x64 else "sdb_masked_dot")
    return out, flag


# ------------------------------------------------------ host-resident batches

_PIPE = {}


def _pipe_streams(dev, ncomp: int = 2):
    s = _PIPE.get((dev.index, ncomp))
    if s is None:  # h2d, d2h, then ncomp compute streams
        s = _PIPE[(dev.index, ncomp)] = tuple(torch.cuda.Stream(dev) for _ in range(2 + ncomp))
    return s


def run_host_batch(fn, host_inputs, host_outputs, device, chunks: int = 8, compute_streams: int = 2):
    """Batched call on HOST-resident (pinned) tensors with the PCIe copies
    overlapped: the batch is cut into `chunks` slices along the leading
    (instance) axis; slice k's host->device copy, slice k-1's kernels and
    slice k-2's device->host copy run concurrently (one copy stream per
    direction -- PCIe is full duplex -- and `compute_streams` compute
    streams, since a slice's grid is smaller than the GPU and latency-bound
    slice kernels overlap).  `chunks` is a slice count or a
    list of slice sizes (a short last slice shortens the D2H tail).  `fn(*device_inputs)` returns the
    device outputs (None entries skipped) matching `host_outputs`.  The
    current stream waits for the last copy, so an event recorded after this
    call covers the whole request."""
    cur = torch.cuda.current_stream(device)
    h2d, d2h, *comps = _pipe_streams(device, max(1, int(compute_streams)))
    for s in (h2d, d2h, *comps):
        s.wait_stream(cur)
    B = host_inputs[0].shape[0]
    if isinstance(chunks, (list, tuple)):  # explicit slice sizes (e.g. a short last slice)
        assert sum(chunks) == B, "slice sizes must cover the batch"
        bounds = [0]
        for c in chunks:
            bounds.append(bounds[-1] + int(c))
    else:
        nch = max(1, min(int(chunks), B))
        bounds = [(B * k) // nch for k in range(nch + 1)]
    chunks = len(bounds) - 1
    for k in range(chunks):
        lo, hi = bounds[k], bounds[k + 1]
        comp = comps[k % len(comps)]
        with torch.cuda.stream(h2d):
            dev_in = [t[lo:hi].to(device, non_blocking=True) for t in host_inputs]
        comp.wait_stream(h2d)
        with torch.cuda.stream(comp):
            outs = [o for o in fn(*dev_in) if o is not None]
        for t in dev_in:
            t.record_stream(comp)
        d2h.wait_stream(comp)
        with torch.cuda.stream(d2h):
            for h, o in zip(host_outputs, outs):
                h[lo:hi].copy_(o, non_blocking=True)
        for o in outs:
            o.record_stream(d2h)
    cur.wait_stream(d2h)
    return host_outputs
