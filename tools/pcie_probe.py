"""Dev utility: PCIe copy timings (pinned) and the pipelined host batch for C2a."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K
dev = torch.device("cuda", 0)
th = torch.randn(256, 513, 129, 3, device=dev)
th[:, 0, :, 0] = float("-inf"); th[:, 0, :, 1] = float("-inf"); th[:, :, 0, 0] = float("-inf"); th[:, :, 0, 2] = float("-inf")
hin = th.cpu().pin_memory()
hout = torch.empty(th.shape, pin_memory=True)
hz = torch.empty(256, dtype=torch.float64, pin_memory=True)
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    w0 = time.perf_counter(); e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it, (time.perf_counter() - w0) * 1e3 / it
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("h2d 203MB   ms (event, wall)", t(lambda: hin.to(dev, non_blocking=True)))
print("d2h 203MB   ms", t(lambda: hout.copy_(th, non_blocking=True)))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): a = hin.to(dev, non_blocking=True)
    with torch.cuda.stream(s2): hout.copy_(th, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
print("h2d||d2h    ms", t(both))
print("kernel      ms", t(lambda: K.nw_fb(th)))
for ch in (1, 2, 4, 8, 16):
    print("pipelined chunks=%2d ms" % ch, t(lambda: K.run_host_batch(lambda x: K.nw_fb(x)[:2], [hin], [hz, hout], dev, chunks=ch)))
for sizes in ([16] * 16, [32] * 7 + [24, 8], [16] * 14 + [24, 8], [8] * 4 + [16] * 14):
    print("pipelined sizes=%s ms" % (sizes[:3],), t(lambda: K.run_host_batch(lambda x: K.nw_fb(x)[:2], [hin], [hz, hout], dev, chunks=sizes)))
