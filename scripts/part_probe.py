"""Partition phase times on the C4 workload (BGMF_PROFILE=1), repeated; with
--once a single partition for an ncu launch list of the radix kernels."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2304_13724_b200 import workloads  # noqa: E402
from paper_2304_13724_b200.device import Engine  # noqa: E402

w = workloads.CONFIGS[os.environ.get("PART_CFG", "C4")]
r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=w.seed)
once = "--once" in sys.argv
os.environ["BGMF_PROFILE"] = "0" if once else "1"
eng = Engine()
for i in range(1 if once else 4):
    t = time.perf_counter()
    eng.partition(r, c, v, w.n, w.m, w.grid, w.grid)
    print(f"partition {i}: {(time.perf_counter() - t) * 1e3:.1f} ms", file=sys.stderr, flush=True)
off = eng.offsets
print("blocks", len(off) - 1, "nnz", int(off[-1]), "min/max block",
      int(np.diff(off).min()), int(np.diff(off).max()), file=sys.stderr)
eng.close()
