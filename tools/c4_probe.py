"""Dev utility: C4 (B=256, n=128) Eisner / Kuhlmann alone, sequential and concurrent."""
import os
import sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from ktime import bench
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
adj = torch.randn(256, 129, 129, device="cuda", generator=g)
adj[:, :, 0] = float("-inf")
i = torch.arange(129, device="cuda")
adj[:, i, i] = float("-inf")
print("eisner alone     %.4f ms" % bench(lambda: K.eisner(adj), iters=10))
print("kuhlmann alone   %.4f ms" % bench(lambda: K.kuhlmann(adj), iters=10))
print("sequential       %.4f ms" % bench(lambda: (K.eisner(adj), K.kuhlmann(adj)), iters=10))
print("concurrent       %.4f ms" % bench(lambda: K.eisner_kuhlmann(adj), iters=10))
