"""Exact mode (fp64, every update in the reference's order) at full size: epoch
time on the GPU (wall of a 3-epoch minus a 1-epoch train_blocked call) and a
bitwise check of the 1-epoch trace and factors against the oracle's C port of
the reference epoch (16 host threads, also timed).  Usage:
python scripts/exact_bench.py [C3 C4 ...]"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402

for name in sys.argv[1:] or ["C3", "C4"]:
    w = workloads.CONFIGS[name]
    r, c, v = workloads.generate(name)
    d = bm.RatingsDataset(w.n, w.m, r, c, v)
    opts = bm.EngineOptions(exact=True)
    walls, res = {}, {}
    for steps in (1, 3, 1, 3):
        cfg = bm.TrainConfig(k=w.k, grid_i=w.grid, grid_j=w.grid, outer_steps=steps,
                             alpha=w.alpha, beta=w.beta, seed=w.seed)
        t = time.perf_counter()
        res[steps] = bm.train_blocked(d, cfg, early_stop=False, options=opts)
        walls[steps] = time.perf_counter() - t
    ep = (walls[3] - walls[1]) / 2
    print(f"{name} exact: {ep * 1e3:.1f} ms/epoch = {w.nnz / ep / 1e6:.1f} M upd/s "
          f"(train_blocked walls 1 epoch {walls[1]:.2f} s, 3 epochs {walls[3]:.2f} s; trace "
          f"seconds {[round(s.seconds, 3) for s in res[3].trace]})", flush=True)
    t = time.perf_counter()
    ou, ov, otr, _ = O.train_blocked(w.n, w.m, r, c, v, k=w.k, alpha=w.alpha, beta=w.beta,
                                     outer_steps=1, grid_i=w.grid, grid_j=w.grid, seed=w.seed,
                                     early_stop=False, nthreads=os.cpu_count() or 1)
    to = time.perf_counter() - t
    g = res[1]
    same = (np.array_equal(g.model.u, ou) and np.array_equal(g.model.v, ov)
            and list(g.trace)[0].train_rmse == otr[0]["train_rmse"])
    print(f"{name} oracle (C port, {os.cpu_count()} threads) 1 epoch incl. partition+init: "
          f"{to:.2f} s; GPU exact epoch bit-identical (U, V, train RMSE): {same} "
          f"[{list(g.trace)[0].train_rmse!r} vs {otr[0]['train_rmse']!r}]", flush=True)
