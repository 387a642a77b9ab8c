"""Top SASS lines by warp-stall samples from an ncu report (source page), with
the stall columns that dominate.  Usage: python scripts/ncu_hot.py rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") or "Stall" in x]
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iall]), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
for n, r in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{n:7d} {100 * n / tot:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:70]}")
