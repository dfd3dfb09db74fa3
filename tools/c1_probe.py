"""Dev utility: C1 timings (fb, viterbi, concurrent request), with and without an L2 flush."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, fl, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(it):
        if fl: flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / it * 1e3
for fl in (False, True):
    print("flush=%d fb %.1f us  vit %.1f us  fb||vit %.1f us  fb;vit %.1f us" % (
        fl, t(lambda: K.chain_fb(init, tr), fl), t(lambda: K.chain_viterbi(init, tr), fl),
        t(lambda: K.chain_fb_viterbi(init, tr), fl), t(lambda: (K.chain_fb(init, tr), K.chain_viterbi(init, tr)), fl)))
