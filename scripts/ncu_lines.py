"""Warp-stall samples per CUDA source line (ncu source page, cuda,sass view).
Usage: python scripts/ncu_lines.py report.ncu-rep [N] [kernel-regex]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
flt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
per = defaultdict(int)
src = {}
line = None
for r in csv.reader(out):
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0].isdigit():
        line = int(r[0])
        src[line] = r[1].strip()
    try:
        per[line] += int(r[4])
    except ValueError:
        pass
tot = sum(per.values()) or 1
print(f"total samples {tot}")
for ln, n in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{n:7d} {100 * n / tot:5.1f}%  L{ln}: {src.get(ln, '')[:90]}")
