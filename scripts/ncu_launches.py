"""Print an ncu --csv launch list (metrics per launch) as one row per launch."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki].split("(")[0][-40:]), {})[r[mi]] = r[vi]
names = sorted({m for v in d.values() for m in v})
print("id kernel " + " ".join(names))
for (i, k), m in d.items():
    print(i, k, " ".join(m.get(n, "") for n in names))
