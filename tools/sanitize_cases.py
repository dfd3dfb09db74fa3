"""Every kernel family at small batch for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck, one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Covers the config-path kernels (chain scan cluster kernel, nw_mitm, CTC
direction + marginal kernels, MTT fp64 pipeline, Eisner linear + Kuhlmann,
Tree-CRF fold/lin/emit, PCFG fast + general, semi-Markov, samplers, CLE)
with B = 2 instances of the config shapes (or smaller where the shape is
the same code path)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from golden import builders as bld  # noqa: E402
from paper_2308_03291_b200 import kernels as K  # noqa: E402

dev = lambda x: torch.as_tensor(x, dtype=torch.float32).cuda()  # noqa: E731
only = sys.argv[1:]


def run(name, fn):
    if only and name not in only:
        return
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


init, tr = bld.batch_chain(0, 2, 128, 32)
run("chain_scan", lambda: K.chain_fb(dev(init), dev(tr)))
run("chain_viterbi", lambda: K.chain_viterbi(dev(init), dev(tr)))
i2, t2 = bld.batch_chain(0, 2, 12, 7)
run("chain_small", lambda: (K.chain_fb(dev(i2), dev(t2)), K.chain_viterbi(dev(i2), dev(t2))))
th = bld.batch_alignment(2, 2, 512, 128)
run("nw_mitm", lambda: K.nw_fb(dev(th)))
run("nw_viterbi", lambda: K.nw_viterbi(dev(bld.batch_alignment(2, 2, 40, 30))))
fp, tg = bld.batch_ctc(3, 2, 128, 64, 32)
run("ctc", lambda: K.ctc_fb(dev(fp), torch.as_tensor(tg, dtype=torch.int32).cuda()))
adj = bld.batch_spanning(6, 2, 128)
run("mtt", lambda: (K.mtt(dev(adj)), K.mtt(dev(adj), True), K.mtt(dev(adj), False, False)))
run("eisner", lambda: K.eisner_kuhlmann(dev(adj)))
run("tree", lambda: (K.tree_fb(dev(bld.batch_tree(4, 2, 64, 32))), K.tree_viterbi(dev(bld.batch_tree(4, 2, 12, 3)))))
r, ru, e = bld.batch_pcfg(5, 2, 16, 32, 32)
run("pcfg", lambda: (K.pcfg_fb(dev(r), dev(ru), dev(e)), K.pcfg_grad(dev(r), dev(ru), dev(e)),
                     K.pcfg_viterbi(dev(r), dev(ru), dev(e))))
r2, ru2, e2 = bld.batch_pcfg(5, 1, 5, 40, 36)
run("pcfg_gen", lambda: (K.pcfg_fb(dev(r2), dev(ru2), dev(e2)), K.pcfg_grad(dev(r2), dev(ru2), dev(e2))))
run("semimarkov", lambda: (K.semimarkov_fb(dev(bld.batch_semi_markov(1, 2, 24, 4, 6))),
                           K.semimarkov_viterbi(dev(bld.batch_semi_markov(1, 2, 24, 4, 6)))))
run("cle", lambda: K.cle(dev(bld.batch_spanning(7, 2, 40))))
th2 = bld.batch_alignment(7, 1, 9, 6)
noise = torch.as_tensor(np.random.default_rng(3).gumbel(size=K.stream_len("alignment", dict(n=9, m=6))))
run("nw_sample", lambda: K.nw_sample(dev(th2), noise[None].cuda(), 1))
print("all ok")
