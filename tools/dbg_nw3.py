"""Dev utility: check the meet-in-the-middle alpha/beta workspace against the oracle."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2308_03291_b200 import _lib
from paper_2308_03291_b200.kernels import ptr, stream_ptr
from golden.builders import batch_alignment
from oracle import sd_oracle as O
lib = _lib.load()
L2E = 1.4426950408889634
B, n, m = 3, 512, 128
NW = (m + 32) // 32
steps = n + 32
th = torch.as_tensor(batch_alignment(1000, B, n, m), dtype=torch.float32).cuda()
t0 = th[0].cpu().numpy().astype(np.float64)
al = O.nw_alpha(t0) * L2E
be = O.nw_beta(t0) * L2E
RF = [(40 * (NW - 1 - 2 * w) + n - 1) >> 1 for w in range(NW)]
for trial in range(1):
    if trial == 1:  # dirty the smem / caches with another kernel family
        x = torch.full((1 << 24,), float("nan"), device="cuda"); del x
    logz = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    marg = torch.full_like(th, float("nan"))
    nb = lib.sdb_nw_fb_workspace(B, n, m)
    ws = torch.full((nb // 4 + 1,), float("nan"), device="cuda")
    rc = lib.sdb_nw_fb(ptr(th), B, n, m, ptr(logz), ptr(marg), ptr(st), ptr(ws), nb, stream_ptr(th.device))
    torch.cuda.synchronize()
    print("rc", rc, "status", st.tolist(), "nb", nb, "logz", logz.tolist(), flush=True)
    w2 = ws[: 2 * B * NW * steps * 32 * 2].view(2, B, NW, steps, 32, 2).cpu().numpy().astype(np.float64)
    wa, wb = w2[0, 0], w2[1, 0]
    ea, eb, na, nb_ = 0.0, 0.0, 0, 0
    for j in range(m + 1):
        w, l = j >> 5, j & 31
        for i in range(n + 1):
            s = i + l
            if i <= RF[w]:
                v = wa[w, s, l, 0] + wa[w, s, l, 1]
                if np.isnan(v): na += 1
                elif np.isfinite(al[i, j]): ea = max(ea, abs(v - al[i, j]))
            else:
                v = wb[w, s, l, 0] + wb[w, s, l, 1]
                if np.isnan(v): nb_ += 1
                elif np.isfinite(be[i, j]): eb = max(eb, abs(v - be[i, j]))
    for w in range(NW):
        miss = {}
        for l in range(32):
            j = 32 * w + l
            if j > m: continue
            rows = [i for i in range(RF[w] + 1) if np.isnan(wa[w, i + l, l, 0])]
            if rows: miss[l] = (len(rows), rows[0], rows[-1])
        print("strip", w, "RF", RF[w], "alpha missing per lane (count, first, last):", dict(list(miss.items())[:6]), "... lanes", len(miss))
        missb = {}
        for l in range(32):
            j = 32 * w + l
            if j > m: continue
            rows = [i for i in range(RF[w] + 1, n + 1) if np.isnan(wb[w, i + l, l, 0])]
            if rows: missb[l] = (len(rows), rows[0], rows[-1])
        print("   beta missing:", dict(list(missb.items())[:6]), "... lanes", len(missb))
    mm = marg[0].cpu().numpy()
    z, mg = O.nw_marginals(t0)
    bad = np.argwhere(np.isnan(mm) | (np.abs(mm - mg) > 1e-4))
    print("trial", trial, "logz err", logz[0].item() - z, "alpha nan", na, "err", ea, "beta nan", nb_, "err", eb,
          "marg bad", len(bad), bad[:6].tolist(), flush=True)
