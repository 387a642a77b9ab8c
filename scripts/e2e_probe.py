"""Phase times of train_blocked (BGMF_PROFILE=1) repeated on the C4 workload,
plus the host's CPU budget (cgroup quota, affinity): the e2e number depends on
host threads for the narrowing upload / widening download."""
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402

for f in ("/sys/fs/cgroup/cpu.max", "/sys/fs/cgroup/cpuset.cpus.effective",
          "/sys/kernel/mm/transparent_hugepage/enabled"):
    try:
        print(f, open(f).read().strip())
    except OSError as e:
        print(f, "n/a", e)
print("affinity", len(os.sched_getaffinity(0)), "cpu_count", os.cpu_count(),
      "OMP_NUM_THREADS", os.environ.get("OMP_NUM_THREADS"))
print(subprocess.run(["uptime"], capture_output=True, text=True).stdout.strip())
w = workloads.CONFIGS["C4"]
t = time.perf_counter()
r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=w.seed)
print(f"gen {time.perf_counter() - t:.1f} s")
d = bm.RatingsDataset(w.n, w.m, r, c, v)
cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, grid_i=w.grid, grid_j=w.grid,
                     seed=w.seed, outer_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 10)
os.environ["BGMF_PROFILE"] = "1"
for i in range(5):
    t = time.perf_counter()
    bm.train_blocked(d, cfg, early_stop=False)
    print(f"run {i}: {time.perf_counter() - t:.3f} s", file=sys.stderr, flush=True)
    print(subprocess.run(["uptime"], capture_output=True, text=True).stdout.strip(), file=sys.stderr)
