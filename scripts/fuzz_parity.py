"""Randomised parity sweep (GPU vs the oracle): random shapes, densities,
duplicates, grids, k and schedules; fast mode within 1e-3 absolute per epoch
(train and test RMSE), exact mode bit-identical; partition arrays bit-equal.
Usage: python scripts/fuzz_parity.py [cases] [seed] [scale] [only-case]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
scale = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # x dims and x^2 ratings
only = int(sys.argv[4]) if len(sys.argv) > 4 else None  # re-run one case (same draws)
fails = 0
t0 = time.time()
for i in range(cases):
    n, m = int(g.integers(1, 3000 * scale)), int(g.integers(1, 3000 * scale))
    nnz = int(min(n * m, g.integers(1, 60_000 * scale * scale)))
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    if g.random() < 0.3 and nnz > 10:  # duplicate cells
        k_ = int(g.integers(1, nnz // 5 + 2))
        src, dst = g.integers(0, nnz, k_), g.integers(0, nnz, k_)
        r[dst], c[dst] = r[src], c[src]
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    I, J = int(g.integers(1, min(n, 20) + 1)), int(g.integers(1, min(m, 20) + 1))
    k = int(g.choice([1, 2, 3, 5, 8, 12, 16, 24, 30, 32, 48, 64, 96, 100, 128]))
    spec = str(g.choice(["const:1", "const:2", "inc:2,3", "dec:3", "adaptive:2",
                         "converge:0.05"]))
    sched = {"const:1": bm.Constant(1), "const:2": bm.Constant(2),
             "inc:2,3": bm.IncreasingEvery(2, 3), "dec:3": bm.Decreasing(3),
             "adaptive:2": bm.AdaptiveDecreasing(2),
             "converge:0.05": bm.ConvergeEachBlock(0.05)}[spec]
    exact = g.random() < 0.25
    # out-of-core: a device budget of a few blocks' ratings (fast mode only)
    stream = (not exact) and g.random() < 0.25 and nnz >= 1000
    steps = int(g.integers(1, 5))
    d = bm.RatingsDataset(n, m, r, c, v)
    holdout = g.random() < 0.3 and nnz >= 20
    tag = f"case {i}: n={n} m={m} nnz={nnz} grid={I}x{J} k={k} {spec} exact={exact} holdout={holdout} stream={stream}"
    if only is not None and i != only:
        continue
    try:
        P = O.partition(r, c, v, n, m, I, J)
        b = bm.partition(d, I, J)
        assert np.array_equal(b._offsets, P["offsets"]) and np.array_equal(b._values,
                                                                           P["values"])
        assert np.array_equal(b._rows, P["rows"]) and np.array_equal(b._cols, P["cols"])
        cfg = bm.TrainConfig(k=k, outer_steps=steps, grid_i=I, grid_j=J, alpha=2e-4,
                             inner_schedule=sched)
        tr, te = bm.split(d, 0.2, seed=i) if holdout else (d, None)
        if holdout:  # the partition above was of the full set; train on the split
            P = None
        opts = None
        if exact:
            opts = bm.EngineOptions(exact=True)
        elif stream:
            per_block = max(1, len(tr) // (I * J))
            opts = bm.EngineOptions(device_rating_budget=12 * 3 * max(per_block * 3, 64))
        try:
            res = bm.train_blocked(tr, cfg, te, early_stop=False, options=opts)
        except Exception as e:  # noqa: BLE001  a slot smaller than the largest block: skip
            if stream and "slot" in str(e):
                continue
            raise
        ou, ov, otr, _ = O.train_blocked(tr.n, tr.m, tr.rows, tr.cols, tr.values, k=k,
                                         outer_steps=steps, grid_i=I, grid_j=J, alpha=2e-4,
                                         schedule=spec, early_stop=False,
                                         test=(te.rows, te.cols, te.values) if holdout else None)
        got = np.array([s.train_rmse for s in res.trace])
        want = np.array([s["train_rmse"] for s in otr])
        if holdout:
            gt = np.array([s.test_rmse for s in res.trace])
            wt = np.array([s["test_rmse"] for s in otr])
            # test RMSE: GPU fp64 reduction vs numpy's pairwise sum (not bit-equal)
            assert (np.all(np.abs(gt - wt) <= 1e-12 * wt) if exact
                    else np.all(np.abs(gt - wt) <= 1e-3)), (gt, wt)
        if exact:
            assert np.array_equal(got, want), (got, want)
            assert np.array_equal(res.model.u, ou) and np.array_equal(res.model.v, ov)
        else:
            assert np.all(np.abs(got - want) <= 1e-3), (np.abs(got - want).max(), got, want)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"FAIL {tag}: {type(e).__name__}: {str(e)[:300]}", flush=True)
print(f"{cases} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
