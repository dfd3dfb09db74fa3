"""Dev utility: Tree-CRF kernel time vs batch size (latency vs throughput)."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from ktime import bench
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
for B in (1, 16, 128, 148, 296, 592):
    th = torch.randn(B, 64, 64, 32, device="cuda", generator=g)
    print("B=%4d fb %.4f ms  logz %.4f ms" % (B, bench(lambda: K.tree_fb(th)), bench(lambda: K.tree_fb(th, marginals=False))))
for n in (8, 16, 32, 64):
    th = torch.randn(128, n, n, 32, device="cuda", generator=g)
    print("n=%3d fb %.4f ms  logz %.4f ms" % (n, bench(lambda: K.tree_fb(th)), bench(lambda: K.tree_fb(th, marginals=False))))
