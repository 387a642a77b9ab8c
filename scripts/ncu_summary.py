"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
--set full capture (.ncu-rep) into a markdown table for profiles/."""

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        out.append(f"\n**{vals[h.index('Kernel Name')].split('(')[0]}**\n")
        out.append("| metric | value | unit |\n|---|---:|---|")
        for m in METRICS:
            if m in h:
                out.append(f"| `{m}` | {vals[h.index(m)]} | {units[h.index(m)]} |")
    return "\n".join(out)


if __name__ == "__main__":
    lst, rep = sys.argv[1], sys.argv[2]
    print("### Launch list (ncu, cold-cache, serialised: compare shares)\n")
    print(launches(lst))
    print("\n### Full capture (`ncu --set full`), one launch per kernel\n")
    print(full(rep))
