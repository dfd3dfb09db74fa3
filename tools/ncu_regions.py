"""Dev utility: stall samples of an ncu report aggregated over SASS address
regions.  Usage: python tools/ncu_regions.py rep.ncu-rep lo:hi:name ... (hex
offsets from the kernel's first instruction)."""
import csv
import subprocess
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb", "stall_math",
           "stall_membar", "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb",
           "stall_wait", "stall_misc"]


def main(rep, regions):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True).stdout.decode("latin-1")
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if "Address" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ia, iall, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = int(data[0][ia], 16)
    tot = sum(float(r[iall] or 0) for r in data)
    agg = {}
    for r in data:
        a = int(r[ia], 16) - base
        name = "other"
        for lo, hi_, nm in regions:
            if lo <= a < hi_:
                name = nm
        d = agg.setdefault(name, {"samples": 0.0, "inst": 0.0})
        d["samples"] += float(r[iall] or 0)
        d["inst"] += float(r[iex] or 0)
        for k in REASONS:
            d[k] = d.get(k, 0.0) + float(r[h.index(k)] or 0)
    for name, d in agg.items():
        st = sorted(((d[k], k[6:]) for k in REASONS), reverse=True)
        print("%-10s %5.1f%% samples, %12.0f warp-inst | %s" % (
            name, 100 * d["samples"] / tot, d["inst"],
            ", ".join("%s %.0f%%" % (n, 100 * v / max(d["samples"], 1)) for v, n in st[:5] if v > 0)))


if __name__ == "__main__":
    regs = []
    for a in sys.argv[2:]:
        lo, hi_, nm = a.split(":")
        regs.append((int(lo, 16), int(hi_, 16), nm))
    main(sys.argv[1], regs)
