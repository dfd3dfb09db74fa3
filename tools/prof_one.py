"""Dev utility: run one kernel family a few times at config shape (for ncu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K

NEG_INF = float("-inf")
fam = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "fb"
g = torch.Generator(device="cuda").manual_seed(0)
if fam == "nw":
    B, n, m = 256, 512, 128
    th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
    th[:, 0, :, 0] = NEG_INF; th[:, 0, :, 1] = NEG_INF; th[:, :, 0, 0] = NEG_INF; th[:, :, 0, 2] = NEG_INF
    fn = {"fb": lambda: K.nw_fb(th), "logz": lambda: K.nw_fb(th, False), "vit": lambda: K.nw_viterbi(th)}[mode]
elif fam in ("chain", "chainv"):
    init = torch.randn(32, 32, device="cuda", generator=g)
    tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
    fn = {"fb": lambda: K.chain_fb(init, tr), "lz": lambda: K.chain_fb(init, tr, False),
          "vit": lambda: K.chain_viterbi(init, tr),
          "both": lambda: K.chain_fb_viterbi(init, tr)}["vit" if fam == "chainv" else mode]
elif fam in ("mtt", "eisner", "kuhl"):
    adj = torch.randn(512 if fam == "mtt" else 256, 129, 129, device="cuda", generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(129, device="cuda")
    adj[:, i, i] = NEG_INF
    fn = {"mtt": lambda: K.mtt(adj), "eisner": lambda: K.eisner(adj), "kuhl": lambda: K.kuhlmann(adj)}[fam]
elif fam == "ctc":
    fp = torch.randn(256, 512, 128, device="cuda", generator=g)
    tg = torch.randint(1, 128, (256, 128), device="cuda", generator=g, dtype=torch.int32)
    fn = lambda: K.ctc_fb(fp, tg)
elif fam == "tree":
    th = torch.randn(128, 64, 64, 32, device="cuda", generator=g)
    fn = lambda: K.tree_fb(th)
elif fam == "pcfg":
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from golden.builders import batch_pcfg
    r, ru, e = batch_pcfg(5000, 128, 64, 32, 32)
    dv = lambda x: torch.as_tensor(x, dtype=torch.float32).cuda()  # noqa: E731
    r, ru, e = dv(r), dv(ru), dv(e)
    fn = lambda: K.pcfg_fb(r, ru, e)
for _ in range(3):
    fn()
torch.cuda.synchronize()
print("ok")
