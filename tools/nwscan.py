import sys, os
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from ktime import bench
from paper_2308_03291_b200 import kernels as K
NEG_INF = float("-inf")
g = torch.Generator(device="cuda").manual_seed(0)
for B in (1, 16, 148, 256, 296, 444, 592):
    n, m = 512, 128
    th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
    th[:, 0, :, 0] = NEG_INF; th[:, 0, :, 1] = NEG_INF; th[:, :, 0, 0] = NEG_INF; th[:, :, 0, 2] = NEG_INF
    print("B=%4d logz %.4f ms  fb %.4f ms" % (B, bench(lambda: K.nw_fb(th, marginals=False)), bench(lambda: K.nw_fb(th))))
for m in (31, 63, 95, 127, 159):
    B, n = 256, 512
    th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
    th[:, 0, :, 0] = NEG_INF; th[:, 0, :, 1] = NEG_INF; th[:, :, 0, 0] = NEG_INF; th[:, :, 0, 2] = NEG_INF
    print("m=%4d logz %.4f ms  fb %.4f ms" % (m, bench(lambda: K.nw_fb(th, marginals=False)), bench(lambda: K.nw_fb(th))))
