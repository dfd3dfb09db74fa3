"""Dev utility: end-to-end (pinned host in/out) timing of one BASELINE config through
kernels.run_host_batch (the bench's e2e path) under slice schedules and compute-stream
counts.  Usage: python tools/e2e_sweep_cfg.py c2b"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2308_03291_b200 import kernels as K

cfg = sys.argv[1]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
inputs = bench.make_inputs(cfg, dev, 0)
fn = bench.step_fn(cfg, inputs)
host_in = [t.cpu().pin_memory() for t in inputs]
probe = [o for o in fn() if o is not None]
host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in probe]
B = host_in[0].shape[0]


def run(chunks, ncomp, reps=12, warm=6):
    ts = []
    for it in range(warm + reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        K.run_host_batch(lambda *d: bench.step_fn(cfg, d)(), host_in, host_out, dev, chunks=chunks,
                         compute_streams=ncomp)
        e1.record()
        torch.cuda.synchronize()
        if it >= warm:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


cur = bench.E2E_CHUNKS.get(cfg, 1)
scheds = [("current", cur), ("1", 1), ("2", 2), ("4", 4), ("8", 8), ("16", 16)]
for name, ch in scheds:
    if isinstance(ch, int) and ch > B:
        continue
    for ncomp in (2, 4):
        t = run(ch, ncomp)
        print("%s %-10s compute_streams=%d  %.3f ms  -> %.0f structures/s" % (cfg, name, ncomp, t, B / t * 1e3),
              flush=True)
