"""Dev utility: per-region stall breakdown from `ncu --page source --csv --print-source sass`.
Usage: python tools/ncu_src.py src.csv [lo:hi:name ...]  (offsets relative to function start, hex)"""
import csv
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb", "stall_math",
           "stall_membar", "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb",
           "stall_wait", "stall_misc"]


def main(path, regions):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = rows[2:]
    ia, iall, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = min(int(r[ia], 16) for r in data)
    tot = sum(float(r[iall] or 0) for r in data)
    agg = {}
    for r in data:
        a = int(r[ia], 16) - base
        name = "other"
        for lo, hi, nm in regions:
            if lo <= a < hi:
                name = nm
        d = agg.setdefault(name, {"samples": 0.0, "inst": 0.0})
        d["samples"] += float(r[iall] or 0)
        d["inst"] += float(r[iex] or 0)
        for k in REASONS:
            d[k] = d.get(k, 0.0) + float(r[h.index(k)] or 0)
    for name, d in agg.items():
        print("%-12s %5.1f%% samples  %.1fM inst  " % (name, 100 * d["samples"] / tot, d["inst"] / 1e6)
              + " ".join("%s=%.0f%%" % (k[6:], 100 * d[k] / max(d["samples"], 1)) for k in REASONS
                         if d[k] > 0.02 * d["samples"]))


if __name__ == "__main__":
    regs = []
    for spec in sys.argv[2:]:
        lo, hi, nm = spec.split(":")
        regs.append((int(lo, 16), int(hi, 16), nm))
    main(sys.argv[1], regs)
