import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2308_03291_b200 import kernels as K
from golden.builders import batch_chain
from oracle import sd_oracle as O
NEG_INF = float("-inf")
init, tr = batch_chain(310, 4, 128, 32)
tr[1] *= 30.0
tr[2, 120, :, 1:] = NEG_INF
tr[3, 5, :, :] -= 200.0
d = lambda x: torch.as_tensor(x, dtype=torch.float32).cuda()
logz, mi, mt, st = K.chain_fb(d(init), d(tr))
for b in range(4):
    z, pi, pt = O.chain_marginals(init[b:b+1], tr[b:b+1])
    e_mi = np.abs(mi[b].cpu().numpy() - pi[0]) / (1e-6 + 1e-4 * np.abs(pi[0]))
    e_mt = np.abs(mt[b].cpu().numpy() - pt[0]) / (1e-6 + 1e-4 * np.abs(pt[0]))
    print(b, "logz", logz[b].item(), z[0], "mi worst (tol units)", e_mi.max(), "mt worst", e_mt.max(), "argmax mi", np.argmax(pi[0]), pi[0].max())
