"""Randomised parity, second sweep: CPMF (train_sync_parallel) shards, early
stopping with random delta, large grids (up to 200 x 200 blocks) and the
block_hook path; GPU vs the oracle.  Usage: python scripts/fuzz_more.py [cases] [seed]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
t0 = time.time()
for i in range(cases):
    n, m = int(g.integers(2, 4000)), int(g.integers(2, 4000))
    nnz = int(min(n * m, g.integers(10, 80_000)))
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    d = bm.RatingsDataset(n, m, r, c, v)
    k = int(g.choice([2, 8, 16, 30, 32, 64, 128]))
    exact = g.random() < 0.3
    opts = bm.EngineOptions(exact=True) if exact else None
    kind = str(g.choice(["cpmf", "early", "biggrid", "hook"]))
    tag = f"case {i}: {kind} n={n} m={m} nnz={nnz} k={k} exact={exact}"
    try:
        if kind == "cpmf":
            wk = int(g.integers(1, 17))
            cfg = bm.TrainConfig(k=k, outer_steps=3, workers=wk, alpha=2e-4)
            res = bm.train_sync_parallel(d, cfg, early_stop=False, options=opts)
            ou, ov, otr, _ = O.train_sync_parallel(n, m, r, c, v, k=k, outer_steps=3,
                                                   workers=wk, alpha=2e-4, early_stop=False)
            tag += f" workers={wk}"
        else:
            if kind == "biggrid":
                I, J = int(g.integers(1, min(n, 200) + 1)), int(g.integers(1, min(m, 200) + 1))
            else:
                I, J = int(g.integers(1, min(n, 16) + 1)), int(g.integers(1, min(m, 16) + 1))
            delta = float(g.choice([1e-2, 1e-3, 0.05])) if kind == "early" else 1e-2
            steps = 30 if kind == "early" else 2
            cfg = bm.TrainConfig(k=k, outer_steps=steps, grid_i=I, grid_j=J, alpha=3e-4,
                                 delta=delta)
            tag += f" grid={I}x{J} delta={delta}"
            hook_calls = []
            hook = (lambda phase, task: hook_calls.append(phase)) if kind == "hook" else None
            res = bm.train_blocked(d, cfg, early_stop=(kind == "early"), options=opts,
                                   block_hook=hook)
            ou, ov, otr, ostop = O.train_blocked(n, m, r, c, v, k=k, outer_steps=steps,
                                                 grid_i=I, grid_j=J, alpha=3e-4, delta=delta,
                                                 early_stop=(kind == "early"))
            if kind == "early":
                assert len(res.trace) == len(otr) or not exact, (len(res.trace), len(otr))
                assert res.stop_reason == ostop or not exact
            if kind == "hook":
                assert hook_calls.count("start") == hook_calls.count("end") > 0
        got = np.array([s.train_rmse for s in res.trace])
        want = np.array([s["train_rmse"] for s in otr])
        if exact:
            assert np.array_equal(got, want), (got, want)
            assert np.array_equal(res.model.u, ou) and np.array_equal(res.model.v, ov)
        else:
            nn = min(len(got), len(want))  # early stop may differ by a step in fast mode
            assert np.all(np.abs(got[:nn] - want[:nn]) <= 1e-3), (np.abs(got[:nn] - want[:nn]).max())
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"FAIL {tag}: {type(e).__name__}: {str(e)[:300]}", flush=True)
print(f"{cases} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
