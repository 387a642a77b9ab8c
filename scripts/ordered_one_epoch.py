"""One C4 epoch forced through the ordered fp32 kernel (for ncu captures)."""
import sys

sys.path.insert(0, ".")
import paper_2304_13724_b200 as bm  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402

w = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
r, c, v = workloads.generate(w.name)
d = bm.RatingsDataset(w.n, w.m, r, c, v)
cfg = bm.TrainConfig(k=w.k, grid_i=w.grid, grid_j=w.grid, outer_steps=2, alpha=w.alpha,
                     beta=w.beta, seed=w.seed)
res = bm.train_blocked(d, cfg, early_stop=False, options=bm.EngineOptions(ordered=True))
print([s.train_rmse for s in res.trace], [round(s.seconds, 4) for s in res.trace])
