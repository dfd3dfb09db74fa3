"""Dev utility: alignment fb with NaN-prefilled outputs / workspace."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2308_03291_b200 import _lib
from paper_2308_03291_b200.kernels import ptr, stream_ptr
from golden.builders import batch_alignment
from oracle import sd_oracle as O
lib = _lib.load()
for (B, n, m) in [(5, 7, 70), (3, 100, 200), (2, 1, 1), (3, 512, 128)]:
    th = torch.as_tensor(batch_alignment(1000, B, n, m), dtype=torch.float32).cuda()
    z, mg = O.nw_marginals(th[0].cpu().numpy().astype(np.float64))
    for fill_marg, fill_ws in [(0, 0), (1, 0), (0, 1)]:
        logz = torch.empty(B, dtype=torch.float64, device="cuda")
        st = torch.empty(B, dtype=torch.int32, device="cuda")
        marg = torch.full_like(th, float("nan") if fill_marg else 0.0)
        nb = lib.sdb_nw_fb_workspace(B, n, m)
        ws = torch.full((nb // 4 + 1,), float("nan") if fill_ws else 0.0, device="cuda")
        rc = lib.sdb_nw_fb(ptr(th), B, n, m, ptr(logz), ptr(marg), ptr(st), ptr(ws), nb, stream_ptr(th.device))
        torch.cuda.synchronize()
        mm = marg[0].cpu().numpy()
        bad = np.argwhere(np.isnan(mm))
        print((B, n, m), "fill", fill_marg, fill_ws, "rc", rc, "nan", len(bad), bad[:5].tolist(), "maxerr",
              float(np.nanmax(np.abs(mm - mg))), flush=True)
