"""Dev utility: tree_fb at B=128, m=32 for n in 8..64 (ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
for n in (8, 16, 32, 64):
    th = torch.randn(128, n, n, 32, device="cuda", generator=g)
    K.tree_fb(th)
torch.cuda.synchronize()
print("ok")
