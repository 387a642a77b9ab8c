"""SM<->L2 ceiling of the sweep's V-row traffic (bgmf_probe_l2) on cuda:0:
random 512 B rows of an L2-resident 17800 x 128 fp32 V (the C4 V block set),
read / read + reduce / reduce / two reads + reduce, and "split-warps": even
warps read + reduce `ratings` rows while odd warps read another `ratings` rows
(a sweep and an SSE co-resident), at 2 and 4 resident 256-thread CTAs per SM."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
from paper_2304_13724_b200 import _native as N  # noqa: E402

L = N.load()
rows, ratings = 17800, 50_000_000
out = {}
for mode, name, bpr in ((0, "read", 512), (1, "read+red", 1024), (2, "red", 512), (3, "2read+red", 1536),
                        (4, "split-warps", 1536)):
    for cps in (2, 4):
        ms = ctypes.c_double()
        N.check(L.bgmf_probe_l2(0, rows, ratings, mode, cps, ctypes.byref(ms)))
        gbs = ratings * bpr / (ms.value / 1e3) / 1e9
        out[f"{name}@{cps}"] = {"ms": ms.value, "GB/s": gbs, "rows/s": ratings / (ms.value / 1e3)}
        print(f"{name:9s} ctas/SM={cps}  {ms.value:8.3f} ms  {gbs:9.1f} GB/s  "
              f"{ratings / (ms.value / 1e3) / 1e9:6.2f} G rows/s", flush=True)
print(json.dumps(out))
