import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2304_13724_b200 as bm
from oracle import oracle as O
for (n, m, k, it) in [(1, 2676, 24, 2), (1, 3000, 128, 1), (2, 2000, 32, 1), (3, 5000, 64, 2)]:
    g = np.random.default_rng(0)
    cells = g.choice(n * m, n * m, replace=False); r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, n * m)), 1, 5)
    d = bm.RatingsDataset(n, m, r, c, v)
    cfg = bm.TrainConfig(k=k, outer_steps=2, grid_i=1, grid_j=1, alpha=2e-4, inner_schedule=bm.Constant(it))
    res = bm.train_blocked(d, cfg, early_stop=False)
    _, _, otr, _ = O.train_blocked(n, m, r, c, v, k=k, outer_steps=2, grid_i=1, grid_j=1, alpha=2e-4, schedule=f"const:{it}", early_stop=False)
    got = np.array([s.train_rmse for s in res.trace]); want = np.array([s["train_rmse"] for s in otr])
    print(n, m, k, it, "drift", np.abs(got - want).max(), "rel", (np.abs(got - want) / want).max())
