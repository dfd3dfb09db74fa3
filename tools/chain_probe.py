"""Dev probe: time the C1 chain kernels alone -- each call captured once in a
CUDA graph and replayed (no host overhead inside the events), after a clock
warm-up; median of per-replay times."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_03291_b200 import kernels as K

g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
fns = {"fb": lambda: K.chain_fb(init, tr), "vit": lambda: K.chain_viterbi(init, tr),
       "both": lambda: K.chain_fb_viterbi(init, tr)}
graphs = {}
for name, fn in fns.items():
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    graphs[name] = gr
t0 = time.time()
while time.time() - t0 < 0.5:
    for gr in graphs.values():
        gr.replay()
torch.cuda.synchronize()
for name, gr in graphs.items():
    ts = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "us median %.1f  min %.1f" % (statistics.median(ts), min(ts)))
