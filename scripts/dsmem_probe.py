"""DSMEM vs L2 for the sweep's V block: one C4 V block
(1113 rows x 128 fp32 = 570 KB) spread over a thread-block cluster's shared
memory, random row reads + lossless fp32 atomic row adds through DSMEM
(bgmf_probe_dsmem), against the L2 probe's read + red.global.add.v4 ceiling
(bgmf_probe_l2 mode 1) on the same rows/s scale."""
import ctypes
import sys

sys.path.insert(0, ".")
from paper_2304_13724_b200 import _native as N  # noqa: E402

L = N.load()
ratings = 20_000_000
ms = ctypes.c_double()
N.check(L.bgmf_probe_l2(0, 17800, ratings, 1, 2, ctypes.byref(ms)))
print(f"L2 read+red.v4 (17800 rows, 2 CTAs/SM)        {ratings / ms.value / 1e6:6.2f} G rows/s")
for cs in (4, 8, 16):
    for mode, name in ((7, "remote read"), (5, "remote read+atomic add"), (6, "own-slice read+atomic add")):
        for cps in (1, 2):
            try:
                N.check(L.bgmf_probe_dsmem(0, 1113, ratings, mode, cs, cps, ctypes.byref(ms)))
                print(f"DSMEM cs={cs:2d} {name:26s} ctas/SM={cps}  {ratings / ms.value / 1e6:6.2f} G rows/s",
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"DSMEM cs={cs} {name} ctas/SM={cps}: {e}", flush=True)
