"""Dev utility: summarise an ncu report (key metrics + stall reasons)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "launch__registers_per_thread", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:80])
        for i, k in enumerate(h):
            if k in KEYS:
                print("  %-70s %s %s" % (k, v[i], u[i]))
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  stalls/issue:", ", ".join("%s %.2f" % (n, x) for x, n in sorted(st, reverse=True) if x > 0.03))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
