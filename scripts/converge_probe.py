"""ConvergeEachBlock on the device: C2 and C3 with
converge:0.05, every per-block loop (sweep, post-sweep SSE, improvement test
against tol, cap) inside one ordered-kernel launch per stratum.  Per-epoch
train RMSE, the step's max inner iterations and capped-block count against
the oracle's fp64 restatement of the reference; GPU step time.
Usage: python scripts/converge_probe.py [C2|C3] [epochs]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
w = workloads.CONFIGS[name]
r, c, v = workloads.generate(name)
d = bm.RatingsDataset(w.n, w.m, r, c, v)
cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, grid_i=w.grid, grid_j=w.grid,
                     seed=w.seed, outer_steps=epochs, inner_schedule=bm.ConvergeEachBlock(tol))
bm.train_blocked(d, bm.TrainConfig(k=w.k, grid_i=w.grid, grid_j=w.grid, outer_steps=1),
                 early_stop=False)  # warm
t0 = time.perf_counter()
res = bm.train_blocked(d, cfg, early_stop=False)
wall = time.perf_counter() - t0
t1 = time.perf_counter()
_, _, otr, _ = O.train_blocked(w.n, w.m, r, c, v, k=w.k, alpha=w.alpha, beta=w.beta,
                               grid_i=w.grid, grid_j=w.grid, seed=w.seed, outer_steps=epochs,
                               schedule=f"converge:{tol}", early_stop=False, nthreads=16)
owall = time.perf_counter() - t1
for s, o in zip(res.trace, otr):
    print(f"{name} step {s.step}: train {s.train_rmse:.6f} (oracle {o['train_rmse']:.6f}, "
          f"|d| {abs(s.train_rmse - o['train_rmse']):.2e}); inner iters max {s.inner_iters} "
          f"(oracle {o['inner_iters']}); capped {s.capped_blocks} (oracle "
          f"{o.get('capped_blocks', '?')}); GPU step {s.seconds * 1e3:.1f} ms", flush=True)
drift = max(abs(s.train_rmse - o["train_rmse"]) for s, o in zip(res.trace, otr))
print(f"{name}: max |d train| {drift:.2e}; train_blocked wall {wall:.2f} s (incl. partition); "
      f"oracle (16 threads) {owall:.1f} s", flush=True)
