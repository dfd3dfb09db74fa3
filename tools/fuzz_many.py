"""Dev utility: the seeded GPU fuzz cases of tests/test_gpu_fuzz.py over many more
seeds (default 150 per family) -- shapes across every kernel-dispatch size class,
random forbidden entries, vacuous instances -- against the float64 oracle.
Prints pass / fail counts per family.  Usage: python tools/fuzz_many.py [seeds]"""
import os
import sys
import traceback
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as F  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 150
cases = [("chain", lambda s: F.test_fuzz_chain(s)), ("alignment", lambda s: F.test_fuzz_alignment(s)),
         ("ctc", lambda s: F.test_fuzz_ctc(s)), ("tree", lambda s: F.test_fuzz_tree(s)),
         ("spanning", lambda s: F.test_fuzz_spanning(s, False)), ("spanning-single", lambda s: F.test_fuzz_spanning(s, True)),
         ("semi_markov", lambda s: F.test_fuzz_semi_markov(s)), ("pcfg", lambda s: F.test_fuzz_pcfg(s))]
total_fail = 0
for name, fn in cases:
    ok, bad = 0, []
    for seed in range(1000, 1000 + N):
        try:
            fn(seed)
            ok += 1
        except Exception:  # noqa: BLE001
            bad.append(seed)
            if len(bad) <= 2:
                traceback.print_exc(limit=1)
    total_fail += len(bad)
    print("%-16s %4d passed  %3d failed  %s" % (name, ok, len(bad), bad[:10]), flush=True)
print("total failures:", total_fail)
