"""CMF (train_sequential = BGMF on a 1x1 grid) on C2-shaped data: the single
block runs through the ordered kernel (one block per stratum); epoch time
against the number of stages (ord_stage_ratings)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2304_13724_b200 as bm  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402

w = workloads.CONFIGS["C2"]
r, c, v = workloads.generate("C2")
d = bm.RatingsDataset(w.n, w.m, r, c, v)
cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, outer_steps=3, grid_i=1, grid_j=1)
for sr in [int(x) for x in (sys.argv[1:] or ["262144", "65536", "16384", "4096"])]:
    import os
    os.environ["BGMF_ENGINE_OPTS"] = f"ord_stage_ratings={sr}"
    bm.train_sequential(d, cfg, early_stop=False, timing=False)
    t0 = time.perf_counter()
    res = bm.train_sequential(d, cfg, early_stop=False, timing=False)
    dt = (time.perf_counter() - t0) / 3
    print(f"CMF C2 ord_stage_ratings={sr}: {dt * 1e3:.1f} ms/epoch, rmse {res.trace.steps[-1].train_rmse:.6f}",
          flush=True)
