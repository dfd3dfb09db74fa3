"""Dev utility: run tree_fb at B=1 and B=128 (n=64, m=32) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
for B in (1, 128):
    th = torch.randn(B, 64, 64, 32, device="cuda", generator=g)
    for _ in range(2):
        K.tree_fb(th)
torch.cuda.synchronize()
print("ok")
