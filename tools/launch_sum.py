"""Dev utility: summarise an ncu --csv launch list (gpu__time_duration.sum per
launch) into a markdown table: kernel, launches, total us, share of the run."""
import csv
import sys
from collections import OrderedDict


def main(path, title):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith("\"")) if r]
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik][:70]
        v = float(r[iv].replace(",", "")) / 1e3  # ns -> us
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    print("## %s\n" % title)
    print("| kernel | launches | total us | median us | share |")
    print("|---|---|---|---|---|")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        s = sorted(v)
        print("| `%s` | %d | %.1f | %.1f | %.1f%% |" % (name, len(v), sum(v), s[len(s) // 2], 100 * sum(v) / tot))
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
