import sys; sys.path.insert(0, ".")
import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads
w = workloads.CONFIGS["C4"]; r, c, v = workloads.generate("C4")
d = bm.RatingsDataset(w.n, w.m, r, c, v)
cfg = bm.TrainConfig(k=w.k, grid_i=w.grid, grid_j=w.grid, outer_steps=1, alpha=w.alpha, beta=w.beta, seed=w.seed)
res = bm.train_blocked(d, cfg, early_stop=False, options=bm.EngineOptions(exact=True))
print([s.train_rmse for s in res.trace])
