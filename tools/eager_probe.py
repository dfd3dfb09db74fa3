import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
for name, fn in (("fb", lambda: K.chain_fb(init, tr)), ("vit", lambda: K.chain_viterbi(init, tr)), ("both", lambda: K.chain_fb_viterbi(init, tr))):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(name, "host us/call %.1f  total us/call %.1f" % ((t1 - t0) / 200 * 1e6, (t2 - t0) / 200 * 1e6))
hin = [init.cpu().pin_memory(), tr.cpu().pin_memory()]
import bench
