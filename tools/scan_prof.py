"""Dev probe: per-phase globaltimer stamps of chain_scan_kernel (debug build
tools/_sdb200_prof.so compiled with -DSDB_SCAN_PROF)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2308_03291_b200 import _lib

_lib.LIB_PATH = os.path.join(ROOT, "tools", "_sdb200_prof.so")
from paper_2308_03291_b200 import kernels as K  # noqa: E402

lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
init = torch.randn(32, 32, device="cuda", generator=g)
tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
for _ in range(5):
    K.chain_fb(init, tr)
torch.cuda.synchronize()
buf = np.zeros((1024, 10), dtype=np.uint64)
lib.sdb_debug_scan_times.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.sdb_debug_scan_times(buf.ctypes.data, buf.nbytes) == 0
t = buf[:256].astype(np.int64)
t0 = t[:, :1]
names = ["start", "prod_begin", "A_done", "clusterA", "B_done", "C_done", "lz_done", "clusterC", "emit_done"]
for i, nm in enumerate(names):
    col = (t[:, i:i+1] - t0)[:, 0]
    ok = t[:, i] > 0
    print("%-10s min %7.2f  med %7.2f  max %7.2f kcyc" % (nm, col[ok].min() / 1e3, np.median(col[ok]) / 1e3,
                                                      col[ok].max() / 1e3))
# per-CTA durations of phases
d = lambda a, b: (t[:, b] - t[:, a]) / 1e3  # noqa: E731
print("A (start->A_done) med/max", np.median(d(0, 2)), d(0, 2).max())
print("wait clusterA med/max", np.median(d(2, 3)), d(2, 3).max())
print("B med/max", np.median(d(3, 4)), d(3, 4).max(), "C", np.median(d(4, 5)), d(4, 5).max())
print("emit med/max", np.median(d(7, 8)), d(7, 8).max())

# isolation: one instance (8 CTAs on 8 SMs, nothing co-resident)
init1, tr1 = init[:1].contiguous(), tr[:1].contiguous()
for _ in range(5):
    K.chain_fb(init1, tr1)
torch.cuda.synchronize()
buf[:] = 0
lib.sdb_debug_scan_times(buf.ctypes.data, buf.nbytes)
t = buf[:8].astype(np.int64)
t0 = t[:, :1]
for i, nm in enumerate(names):
    col = (t[:, i:i+1] - t0)[:, 0]
    print("B=1 %-10s %s" % (nm, " ".join("%6.2f" % (x / 1e3) for x in col)))
print("B=1 C alpha-loop end", " ".join("%6.2f" % ((x - y) / 1e3) for x, y in zip(t[:, 8], t[:, 0])))
print("B=1 C beta-loop end ", " ".join("%6.2f" % ((x - y) / 1e3) for x, y in zip(t[:, 9], t[:, 0])))
