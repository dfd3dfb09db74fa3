"""Dev probe: C1-shaped chain fb for ONE instance (one cluster) -- for ncu source views."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_03291_b200 import kernels as K

g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(1, 32, device="cuda", generator=g)
tr = torch.randn(1, 127, 32, 32, device="cuda", generator=g)
for _ in range(5):
    K.chain_fb(init, tr)
torch.cuda.synchronize()
