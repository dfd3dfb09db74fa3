"""Dev utility: C1 (B=32, n=128, m=32) forward-backward / Viterbi alone, sequential, concurrent."""
import os
import sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from ktime import bench
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
for name, fn in (("fb alone", lambda: K.chain_fb(init, tr)), ("viterbi alone", lambda: K.chain_viterbi(init, tr)),
                 ("sequential", lambda: (K.chain_fb(init, tr), K.chain_viterbi(init, tr))),
                 ("concurrent", lambda: K.chain_fb_viterbi(init, tr))):
    gr = torch.cuda.CUDAGraph()
    fn(); torch.cuda.synchronize()
    with torch.cuda.graph(gr):
        fn()
    print("%-14s graph %.4f ms" % (name, bench(gr.replay, iters=50)))
