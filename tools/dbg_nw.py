"""Dev utility: replay the batched alignment test sequence and report errors."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2308_03291_b200 import kernels as K
from golden.builders import batch_alignment
from oracle import sd_oracle as O
def run(B, n, m, seed=1000, extra=True):
    th = batch_alignment(seed, B, n, m)
    logz, marg, st = K.nw_fb(torch.as_tensor(th).cuda())
    torch.cuda.synchronize()
    z, mg = O.nw_marginals(th[0])
    mm = marg[0].cpu().numpy()
    print((B, n, m), "st", st.tolist(), "dz", logz[0].item() - z, "nan", int(np.isnan(mm).sum()), "maxerr", float(np.nanmax(np.abs(mm - mg))), flush=True)
    if extra:
        K.nw_fb(torch.as_tensor(th).cuda(), marginals=False)
        K.nw_viterbi(torch.as_tensor(th).cuda())
        torch.cuda.synchronize()
for shp in [(3, 512, 128), (4, 40, 31), (2, 33, 32), (5, 7, 70), (2, 1, 1), (3, 100, 200)]:
    run(*shp)
run(5, 7, 70, extra=False)
run(4, 40, 31, extra=False)
run(5, 7, 70, extra=False)
