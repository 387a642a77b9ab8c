"""Randomised bit-exactness of the stateless drop-ins (the reference's numba
boundary, _kernels.py) on the GPU vs the oracle: sgd_block (sweeps and
converge), block_sse, batch_gradient_block -- random block shapes, k, alpha
(including diverging ones), duplicates and empty blocks; results, in-place
factor updates and divergence locations must be identical.
Usage: python scripts/fuzz_kernels.py [cases] [seed]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
t0 = time.time()
for i in range(cases):
    h, w = int(g.integers(1, 300)), int(g.integers(1, 300))
    cnt = int(g.integers(0, min(h * w, 5000) + 1))
    rows = g.integers(0, h, cnt)
    cols = g.integers(0, w, cnt)
    vals = np.clip(np.rint(3 + g.normal(0, 1.2, cnt)), 1, 5)
    k = int(g.integers(1, 140))
    alpha = float(g.choice([1e-4, 1e-3, 1e-2, 0.5, 50.0]))
    beta = float(g.choice([0.0, 1e-2, 0.5]))
    u0 = g.random((h, k)) / np.sqrt(k)
    v0 = g.random((w, k)) / np.sqrt(k)
    kind = str(g.choice(["sweeps", "converge", "sse", "gradient"]))
    iters = int(g.integers(1, 4))
    tag = f"case {i}: {kind} h={h} w={w} cnt={cnt} k={k} alpha={alpha} beta={beta} iters={iters}"
    try:
        u1, v1, u2, v2 = u0.copy(), v0.copy(), u0.copy(), v0.copy()
        if kind == "sse":
            task = bm.BlockTask(0, 0, rows, cols, vals, u1, v1, alpha, beta, 1)
            assert bm.block_sse(task) == O.block_sse(rows, cols, vals, u2, v2)
            continue
        if kind == "gradient":
            task = bm.BlockTask(0, 0, rows, cols, vals, u1, v1, alpha, beta, iters)
            try:
                st = bm.batch_gradient_block(task)
                got = (st.sse_before, st.sse_after, -1, -1)
            except bm.DivergenceError as e:
                got = ("div", e.entry, e.iteration)
            ref = O.gradient_steps(rows, cols, vals, u2, v2, alpha, beta, iters)
        elif kind == "converge":
            tol = float(g.choice([1e-2, 1e-4]))
            task = bm.BlockTask(0, 0, rows, cols, vals, u1, v1, alpha, beta, None, tol)
            try:
                st = bm.sgd_block(task)
                got = (st.sse_before, st.sse_after, st.iters_used, int(st.capped), -1, -1)
            except bm.DivergenceError as e:
                got = ("div", e.entry, e.iteration)
            from paper_2304_13724_b200.kernel import CONVERGE_CAP
            ref = O.sgd_converge(rows, cols, vals, u2, v2, alpha, beta, tol, CONVERGE_CAP)
        else:
            task = bm.BlockTask(0, 0, rows, cols, vals, u1, v1, alpha, beta, iters)
            try:
                st = bm.sgd_block(task)
                got = (st.sse_before, st.sse_after, -1, -1)
            except bm.DivergenceError as e:
                got = ("div", e.entry, e.iteration)
            ref = O.sgd_sweeps(rows, cols, vals, u2, v2, alpha, beta, iters)
        if got[0] == "div":  # reference: (.., nan, bad_entry, bad_iter)
            assert ref[-2] == got[1] and ref[-1] == got[2], (got, ref)
        else:
            assert ref[-2] == -1 and tuple(got[:-2]) == tuple(ref[:-2]), (got, ref)
            assert np.array_equal(u1, u2) and np.array_equal(v1, v2)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"FAIL {tag}: {type(e).__name__}: {str(e)[:300]}", flush=True)
print(f"{cases} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
