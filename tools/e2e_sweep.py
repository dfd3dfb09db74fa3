"""Dev utility: C2a end-to-end (pinned host in/out) timing of
kernels.run_host_batch under different instance-slice schedules."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K

NEG_INF = float("-inf")
B, n, m = 256, 512, 128
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)
th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
th[:, 0, :, 0] = NEG_INF; th[:, 0, :, 1] = NEG_INF; th[:, :, 0, 0] = NEG_INF; th[:, :, 0, 2] = NEG_INF
host_in = [th.cpu().pin_memory()]
lz, mg, st = K.nw_fb(th)
host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in (lz, mg, st)]


def run(chunks, reps=15, warm=8):
    fn = lambda t: K.nw_fb(t)  # noqa: E731
    ts = []
    for it in range(warm + reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        K.run_host_batch(fn, host_in, host_out, dev, chunks=chunks)
        e1.record()
        torch.cuda.synchronize()
        if it >= warm:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


scheds = {
    "cur [32]*7+[24,8]": [32] * 7 + [24, 8],
    "[8,24]+[32]*6+[24,8]": [8, 24] + [32] * 6 + [24, 8],
    "[8,8,16]+[32]*6+[16,8,8]": [8, 8, 16] + [32] * 6 + [16, 8, 8],
    "[16]*16": [16] * 16,
    "[8]*32": [8] * 32,
    "[4,12,16]+[32]*6+[16,8,4,4]": [4, 12, 16] + [32] * 6 + [16, 8, 4, 4],
}
for name, c in scheds.items():
    ms = run(c)
    print("%-32s %.3f ms  %.0f structures/s" % (name, ms, B / ms * 1e3))
# copy floor: both directions concurrently, no kernels
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dmg = torch.empty_like(mg)
dth = torch.empty_like(th)
for it in range(10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        dth.copy_(host_in[0], non_blocking=True)
    with torch.cuda.stream(s2):
        host_out[1].copy_(dmg, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
print("copy floor (H2D || D2H, 203 MB each) %.3f ms" % e0.elapsed_time(e1))

# pipeline without the alignment kernel (outputs = preallocated device tensors of the same shapes)
dz, dm, ds = torch.zeros_like(lz), torch.zeros_like(mg), torch.zeros_like(st)


def fake(t):
    b = t.shape[0]
    return dz[:b], dm[:b], ds[:b]


for name, c in (("fake-kernel cur", [32] * 7 + [24, 8]), ("fake-kernel [16]*16", [16] * 16)):
    ts = []
    for it in range(20):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        K.run_host_batch(fake, host_in, host_out, dev, chunks=c)
        e1.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print("%-32s %.3f ms" % (name, ts[len(ts) // 2]))
# per-chunk timeline of the current schedule
c = [32] * 7 + [24, 8]
h2d, d2h, c0, c1 = K._pipe_streams(dev)
torch.cuda.synchronize()
ev = []
t0 = torch.cuda.Event(True); t0.record()
cur = torch.cuda.current_stream()
for s in (h2d, d2h, c0, c1):
    s.wait_stream(cur)
lo = 0
for k, sz in enumerate(c):
    hi = lo + sz
    comp = c0 if k % 2 == 0 else c1
    with torch.cuda.stream(h2d):
        din = host_in[0][lo:hi].to(dev, non_blocking=True)
        a = torch.cuda.Event(True); a.record(h2d)
    comp.wait_stream(h2d)
    with torch.cuda.stream(comp):
        outs = K.nw_fb(din)
        bk = torch.cuda.Event(True); bk.record(comp)
    d2h.wait_stream(comp)
    with torch.cuda.stream(d2h):
        for h, o in zip(host_out, outs):
            h[lo:hi].copy_(o, non_blocking=True)
        cd = torch.cuda.Event(True); cd.record(d2h)
    ev.append((a, bk, cd))
    lo = hi
torch.cuda.synchronize()
for k, (a, bk, cd) in enumerate(ev):
    print("chunk %d: h2d done %.3f  kernel done %.3f  d2h done %.3f" % (k, t0.elapsed_time(a), t0.elapsed_time(bk), t0.elapsed_time(cd)))
