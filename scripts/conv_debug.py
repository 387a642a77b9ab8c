import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads
r, c, v = workloads.lowrank(6040, 3706, 300_000, seed=21)
d = bm.RatingsDataset(6040, 3706, r, c, v)
for g in (0, 1):
    e = bm.Engine(bm.EngineOptions())
    e._opt("conv_graph", float(g))
    e.partition(d.rows, d.cols, d.values, d.n, d.m, 8, 8)
    e.init_factors(d.n, d.m, 32, 0)
    ids, off = e.plan_arrays(bm.plan_step(8, 8, 0))
    sse, iters, capped, bad = e.run_step_converge(ids, off, 0.05, 10000, 1e-4, 1e-2)
    print("graph" if g else "host ", "iters", iters[ids][:16], "sse", np.round(sse[ids][:4], 3), bad)
    e.close()
