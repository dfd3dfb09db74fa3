"""Dev probe: time the C1 chain kernels alone (CUDA events) and report how many
instances took the log-space fallback."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_03291_b200 import kernels as K

g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
for name, fn in (("fb", lambda: K.chain_fb(init, tr)), ("vit", lambda: K.chain_viterbi(init, tr))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, "us per call", e0.elapsed_time(e1) / 20 * 1e3)
