"""Dev utility: CUDA-event timing of the batched kernels at BASELINE config
shapes (device-resident inputs).  Usage: python tools/timeit.py [family ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_03291_b200 import kernels as K

NEG_INF = float("-inf")


def bench(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main(fams):
    g = torch.Generator(device="cuda").manual_seed(0)
    if "chain" in fams:
        init = torch.randn(32, 32, device="cuda", generator=g)
        tr = torch.randn(32, 127, 32, 32, device="cuda", generator=g)
        print("chain_fb      B=32 n=128 m=32  ms %.4f" % bench(lambda: K.chain_fb(init, tr)))
        print("chain_viterbi B=32 n=128 m=32  ms %.4f" % bench(lambda: K.chain_viterbi(init, tr)))
    if "nw" in fams:
        B, n, m = 256, 512, 128
        th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
        th[:, 0, :, 0] = NEG_INF; th[:, 0, :, 1] = NEG_INF; th[:, :, 0, 0] = NEG_INF; th[:, :, 0, 2] = NEG_INF
        t = bench(lambda: K.nw_fb(th))
        print("nw_fb   B=256 512x128 ms %.4f  -> %.1f GB/s algorithmic" % (t, 2 * th.numel() * 4 / t / 1e6))
        print("nw_logz B=256 512x128 ms %.4f" % bench(lambda: K.nw_fb(th, marginals=False)))
        print("nw_viterbi B=256 512x128 ms %.4f" % bench(lambda: K.nw_viterbi(th), iters=5))




def ctc():
    g = torch.Generator(device="cuda").manual_seed(0)
    B, T, V, L = 256, 512, 128, 128
    fp = torch.randn(B, T, V, device="cuda", generator=g)
    tg = torch.randint(1, V, (B, L), device="cuda", generator=g, dtype=torch.int32)
    t = bench(lambda: K.ctc_fb(fp, tg))
    print("ctc_fb  B=256 T=512 V=128 L=128 ms %.4f -> %.0f struct/s" % (t, B / t * 1e3))
    print("ctc_logz ms %.4f" % bench(lambda: K.ctc_fb(fp, tg, False)))
    print("ctc_viterbi ms %.4f" % bench(lambda: K.ctc_viterbi(fp, tg), iters=5))



def tree():
    g = torch.Generator(device="cuda").manual_seed(0)
    th = torch.randn(128, 64, 64, 32, device="cuda", generator=g)
    t = bench(lambda: K.tree_fb(th))
    print("tree_fb B=128 n=64 m=32 ms %.4f -> %.0f struct/s, %.0f GB/s alg" % (t, 128 / t * 1e3, 128 * 790532 / t / 1e6))
    print("tree_logz ms %.4f" % bench(lambda: K.tree_fb(th, False)))
    print("tree_viterbi ms %.4f" % bench(lambda: K.tree_viterbi(th)))



def mtt():
    g = torch.Generator(device="cuda").manual_seed(0)
    adj = torch.randn(512, 129, 129, device="cuda", generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(129, device="cuda")
    adj[:, i, i] = NEG_INF
    t = bench(lambda: K.mtt(adj))
    print("mtt B=512 n=128 ms %.4f -> %.0f struct/s, %.1f TFLOP/s alg" % (t, 512 / t * 1e3, 512 * 4194304 / t / 1e9))
    print("mtt logz ms %.4f" % bench(lambda: K.mtt(adj, marginals=False)))
    print("mtt single-root ms %.4f" % bench(lambda: K.mtt(adj, True)))



def eisner():
    g = torch.Generator(device="cuda").manual_seed(0)
    adj = torch.randn(256, 129, 129, device="cuda", generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(129, device="cuda")
    adj[:, i, i] = NEG_INF
    t = bench(lambda: K.eisner(adj), iters=5)
    print("eisner B=256 n=128 ms %.4f -> %.0f struct/s" % (t, 256 / t * 1e3))
    print("eisner logz ms %.4f" % bench(lambda: K.eisner(adj, marginals=False), iters=5))
    print("kuhlmann ms %.4f" % bench(lambda: K.kuhlmann(adj), iters=5))



def pcfg():
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from golden.builders import batch_pcfg
    root, rules, emis = batch_pcfg(5000, 128, 64, 32, 32)
    dv = lambda x: torch.as_tensor(x, dtype=torch.float32).cuda()  # noqa: E731
    root, rules, emis = dv(root), dv(rules), dv(emis)
    t = bench(lambda: K.pcfg_fb(root, rules, emis), iters=3, warm=1)
    print("pcfg B=128 n=64 NT=PT=32 ms %.3f -> %.0f struct/s" % (t, 128 / t * 1e3))
    print("pcfg logz ms %.3f" % bench(lambda: K.pcfg_fb(root, rules, emis, marginals=False), iters=3, warm=1))


if __name__ == "__main__":
    fams = sys.argv[1:] or ["chain", "nw", "ctc"]
    main(fams)
    for f in fams:
        if f in globals() and f not in ("main", "bench"):
            globals()[f]()
