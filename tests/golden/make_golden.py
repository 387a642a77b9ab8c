"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every number stored here comes from the unmodified reference
(`blockmf` 0.1.0, /root/reference/pkg/src).  The fixtures pin
(a) the CPU oracle (oracle/), which must reproduce them bit-for-bit, and
(b) the GPU path, which must reproduce the integer ones bit-for-bit (partition,
plans) and the floating-point ones within the stated tolerances -- or bit-for-bit
in exact (fp64 sequential) mode.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

import blockmf as bm  # noqa: E402
from blockmf import _kernels  # noqa: E402
from conftest import make_ml100k_standin  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def dense(n):
    return bm.gen_synthetic(bm.SyntheticSpec(n, n, 1, 30, seed=0))


def kernel_cases():
    """sgd_sweeps / block_sse / sgd_converge on random small blocks."""
    rng = np.random.default_rng(2024)
    cases = {}
    for t in range(12):
        h = int(rng.integers(1, 20))
        w = int(rng.integers(1, 20))
        k = int(rng.choice([1, 2, 3, 4, 5, 8, 13, 30, 32]))
        cnt = int(rng.integers(0, h * w + 1))
        cells = np.sort(rng.choice(h * w, size=cnt, replace=False))
        rows, cols = cells // w, cells % w
        vals = rng.integers(1, 6, cnt).astype(np.float64)
        u = rng.random((h, k)) / np.sqrt(k)
        v = rng.random((w, k)) / np.sqrt(k)
        alpha = float(rng.choice([1e-4, 1e-3, 1e-2, 5e-2]))
        beta = float(rng.choice([0.0, 1e-2, 0.1, 0.5]))
        iters = int(rng.integers(1, 5))
        u1, v1 = u.copy(), v.copy()
        sb, sa, be, bi = _kernels.sgd_sweeps(rows, cols, vals, u1, v1, alpha, beta, iters)
        u2, v2 = u.copy(), v.copy()
        tol = 1e-3
        csb, csa, cit, ccap, cbe, cbi = _kernels.sgd_converge(
            rows, cols, vals, u2, v2, alpha, beta, tol, 10_000)
        p = f"c{t}_"
        cases.update({
            p + "rows": rows, p + "cols": cols, p + "vals": vals, p + "u": u, p + "v": v,
            p + "params": np.array([alpha, beta, iters, tol]),
            p + "u_after": u1, p + "v_after": v1,
            p + "out": np.array([sb, sa, be, bi], dtype=np.float64),
            p + "u_conv": u2, p + "v_conv": v2,
            p + "out_conv": np.array([csb, csa, cit, ccap, cbe, cbi], dtype=np.float64),
        })
    # divergence: reference test_kernel.py:119-135 shape
    d32 = dense(32)
    blk = bm.partition(d32, 2, 2).block(1, 0)
    model = bm.init_factors(32, 32, 4, seed=0)
    u = model.u[blk.row_start:blk.row_stop].copy()
    v = model.v[blk.col_start:blk.col_stop].copy()
    sb, sa, be, bi = _kernels.sgd_sweeps(blk.rows, blk.cols, blk.values, u, v, 1e6, 0.0, 50)
    cases["div_out"] = np.array([sb, sa, be, bi], dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "kernel_cases.npz"), n_cases=12, **cases)


def partition_cases():
    out = {}
    meta = {}
    d32 = dense(32)
    rng = np.random.default_rng(7)
    # sparse with empty blocks and unsorted input order
    n, m = 50, 37
    cells = rng.choice(n * m, size=300, replace=False)
    sp = bm.RatingsDataset(n, m, cells // m, cells % m, rng.integers(1, 6, 300))
    # duplicated cells (not validated by partition): lexsort keeps input order
    dup_rows = np.array([3, 1, 3, 3, 0, 1, 3])
    dup_cols = np.array([2, 0, 2, 1, 4, 0, 2])
    dup = bm.RatingsDataset(5, 5, dup_rows, dup_cols, np.arange(7, dtype=float))
    sets = {
        "d32_3x5": (d32, 3, 5),
        "d32_4x4": (d32, 4, 4),
        "sparse_6x5": (sp, 6, 5),
        "sparse_1x1": (sp, 1, 1),
        "dup_2x2": (dup, 2, 2),
        "six_3x3": (bm.RatingsDataset.from_triples(6, 6, [(0, 0, 1.0), (5, 5, 2.0)]), 3, 3),
    }
    for name, (d, gi, gj) in sets.items():
        b = bm.partition(d, gi, gj)
        out[name + "_in_rows"] = d.rows
        out[name + "_in_cols"] = d.cols
        out[name + "_in_vals"] = d.values
        out[name + "_offsets"] = b._offsets
        out[name + "_rows"] = b._rows
        out[name + "_cols"] = b._cols
        out[name + "_vals"] = b._values
        meta[name] = dict(n=d.n, m=d.m, I=gi, J=gj)
    np.savez_compressed(os.path.join(OUT, "partition_cases.npz"), **out)
    # C1 standin: hashes only (100k entries)
    r, c, v = make_ml100k_standin()
    sd = bm.RatingsDataset(943, 1682, r, c, v)
    big = {}
    for gi, gj in ((4, 4), (8, 8), (3, 7)):
        b = bm.partition(sd, gi, gj)
        big[f"{gi}x{gj}"] = dict(
            offsets=sha(b._offsets), rows=sha(b._rows), cols=sha(b._cols),
            values=sha(b._values), counts=b.counts.tolist())
    meta["standin"] = dict(in_rows=sha(sd.rows), in_cols=sha(sd.cols),
                           in_vals=sha(sd.values), partitions=big)
    d64 = dense(64)
    meta["dense64"] = dict(rows=sha(d64.rows), cols=sha(d64.cols), vals=sha(d64.values))
    meta["dense32"] = dict(rows=sha(d32.rows), cols=sha(d32.cols), vals=sha(d32.values))
    d256 = dense(256)
    meta["dense256"] = dict(rows=sha(d256.rows), cols=sha(d256.cols), vals=sha(d256.values))
    tr, te = bm.split(sd, 0.2, seed=0)
    meta["standin_split"] = dict(train_rows=sha(tr.rows), train_cols=sha(tr.cols),
                                 train_vals=sha(tr.values), test_rows=sha(te.rows),
                                 test_cols=sha(te.cols), test_vals=sha(te.values))
    sp2 = bm.gen_synthetic(bm.SyntheticSpec(40, 30, 1, 5, seed=3, density=0.3))
    meta["sparse_gen"] = dict(rows=sha(sp2.rows), cols=sha(sp2.cols), vals=sha(sp2.values),
                              n=len(sp2))
    init = bm.init_factors(943, 1682, 30, 0)
    meta["init_943_1682_30_0"] = dict(u=sha(init.u), v=sha(init.v))
    return meta


def plans():
    res = {}
    for gi in range(1, 9):
        for gj in range(1, 9):
            for step in (0, 1, 2, 5, 9):
                res[f"{gi},{gj},{step}"] = bm.format_plan(bm.plan_step(gi, gj, step))
    return res


def traces():
    out = {}
    meta = {}

    def record(name, d, cfg, test=None, early_stop=False):
        res = bm.train_blocked(d, cfg, test, early_stop=early_stop, timing=False)
        meta[name] = dict(
            train=[s.train_rmse for s in res.trace],
            test=[s.test_rmse for s in res.trace],
            inner=[s.inner_iters for s in res.trace],
            capped=[s.capped_blocks for s in res.trace],
            stop=res.stop_reason,
            final_rmse=bm.rmse(res.model, d),
            u_sha=sha(res.model.u), v_sha=sha(res.model.v),
            cfg=dict(k=cfg.k, alpha=cfg.alpha, beta=cfg.beta, delta=cfg.delta,
                     outer_steps=cfg.outer_steps,
                     schedule=bm.format_schedule(cfg.inner_schedule),
                     grid_i=cfg.grid_i, grid_j=cfg.grid_j, seed=cfg.seed),
            early_stop=early_stop,
        )
        return res

    def cfg64(**kw):
        base = dict(k=10, alpha=1e-4, beta=1e-2, delta=1e-2, seed=0, outer_steps=10,
                    inner_schedule=bm.Constant(1), grid_i=4, grid_j=4)
        base.update(kw)
        return bm.TrainConfig(**base)

    d64 = dense(64)
    r = record("dense64_const1", d64, cfg64())
    out["dense64_const1_u"] = r.model.u
    out["dense64_const1_v"] = r.model.v
    record("dense64_const3", d64, cfg64(inner_schedule=bm.Constant(3), outer_steps=3))
    record("dense64_dec4", d64, cfg64(inner_schedule=bm.Decreasing(4), outer_steps=6))
    record("dense64_inc", d64, cfg64(inner_schedule=bm.IncreasingEvery(2, 3), outer_steps=6))
    record("dense64_adaptive", d64, cfg64(alpha=1e-3, inner_schedule=bm.AdaptiveDecreasing(8),
                                          outer_steps=8))
    record("dense64_converge", d64, cfg64(inner_schedule=bm.ConvergeEachBlock(0.5),
                                          outer_steps=2))
    record("dense64_early", d64, cfg64(outer_steps=100), early_stop=True)
    record("dense64_wide_2x5", d64, cfg64(grid_i=2, grid_j=5, outer_steps=4))
    record("dense64_tall_5x2", d64, cfg64(grid_i=5, grid_j=2, outer_steps=4))
    tr, te = bm.split(d64, 0.2, seed=1)
    record("dense64_holdout", tr, cfg64(outer_steps=3), te)

    r, c, v = make_ml100k_standin()
    sd = bm.RatingsDataset(943, 1682, r, c, v)
    c1 = bm.TrainConfig(k=30, alpha=1e-4, beta=1e-2, delta=1e-2, seed=0, outer_steps=20,
                        grid_i=4, grid_j=4)
    record("c1_k30", sd, c1)
    record("c1_k10", sd, bm.TrainConfig(k=10, outer_steps=10, grid_i=4, grid_j=4))
    tr, te = bm.split(sd, 0.2, seed=0)
    record("c1_split", tr, bm.TrainConfig(k=30, outer_steps=10, grid_i=4, grid_j=4), te)
    np.savez_compressed(os.path.join(OUT, "train_cases.npz"), **out)
    return meta


def baseline_cases():
    """Verification kernels and the baseline trainers:
    _kernels.gradient_steps (_kernels.py:103-140), kernel.block_objective /
    block_gradients (kernel.py:161-179), baselines.train_sequential (CMF) and
    train_sync_parallel (CPMF) (baselines.py:62-182)."""
    rng = np.random.default_rng(2025)
    out = {}
    meta = {"n_grad": 12, "n_obj": 6, "traces": {}}
    for t in range(12):
        h = int(rng.integers(1, 20))
        w = int(rng.integers(1, 20))
        k = int(rng.choice([1, 2, 3, 4, 5, 8, 13, 30, 32, 64]))
        cnt = int(rng.integers(0, h * w + 1))
        cells = np.sort(rng.choice(h * w, size=cnt, replace=False))
        rows, cols = cells // w, cells % w
        vals = rng.integers(1, 6, cnt).astype(np.float64)
        u = rng.random((h, k)) / np.sqrt(k)
        v = rng.random((w, k)) / np.sqrt(k)
        alpha = float(rng.choice([1e-4, 1e-3, 1e-2, 5e-2]))
        beta = float(rng.choice([0.0, 1e-2, 0.1, 0.5]))
        iters = int(rng.integers(1, 5))
        u1, v1 = u.copy(), v.copy()
        sb, sa, be, bi = _kernels.gradient_steps(rows, cols, vals, u1, v1, alpha, beta, iters)
        p = f"g{t}_"
        out.update({p + "rows": rows, p + "cols": cols, p + "vals": vals, p + "u": u, p + "v": v,
                    p + "params": np.array([alpha, beta, iters]), p + "u_after": u1,
                    p + "v_after": v1, p + "out": np.array([sb, sa, be, bi], np.float64)})
    d32 = dense(32)
    blk = bm.partition(d32, 1, 1).block(0, 0)
    model = bm.init_factors(32, 32, 4, seed=0)
    u, v = model.u.copy(), model.v.copy()
    out["gdiv_out"] = np.array(_kernels.gradient_steps(blk.rows, blk.cols, blk.values, u, v,
                                                       1e6, 0.0, 50), np.float64)
    for t in range(6):
        k = int(rng.integers(1, 6))
        nr, nc = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        count = int(rng.integers(1, nr * nc + 1))
        cells = rng.choice(nr * nc, size=count, replace=False)
        task = bm.BlockTask(bi=0, bj=0, rows=cells // nc, cols=cells % nc,
                            values=rng.uniform(1.0, 5.0, count),
                            u_slice=rng.uniform(0.1, 1.0, (nr, k)),
                            v_slice=rng.uniform(0.1, 1.0, (nc, k)), alpha=1e-3,
                            beta=float(rng.uniform(0.0, 0.5)), inner_iters=1)
        gu, gv = bm.block_gradients(task)
        p = f"o{t}_"
        out.update({p + "rows": task.rows, p + "cols": task.cols, p + "vals": task.values,
                    p + "u": task.u_slice, p + "v": task.v_slice, p + "beta": np.array([task.beta]),
                    p + "obj": np.array([bm.block_objective(task)]), p + "gu": gu, p + "gv": gv})

    def rec(name, fn, d, cfg, test=None, early_stop=False, keep=False):
        res = fn(d, cfg, test, early_stop=early_stop, timing=False)
        meta["traces"][name] = dict(
            train=[s.train_rmse for s in res.trace], test=[s.test_rmse for s in res.trace],
            inner=[s.inner_iters for s in res.trace], stop=res.stop_reason,
            u_sha=sha(res.model.u), v_sha=sha(res.model.v),
            cfg=dict(k=cfg.k, alpha=cfg.alpha, beta=cfg.beta, delta=cfg.delta,
                     outer_steps=cfg.outer_steps, seed=cfg.seed, workers=cfg.workers,
                     grid_i=cfg.grid_i, grid_j=cfg.grid_j,
                     schedule=bm.format_schedule(cfg.inner_schedule)),
            early_stop=early_stop)
        if keep:
            out[name + "_u"] = res.model.u
            out[name + "_v"] = res.model.v

    d64 = dense(64)
    base = dict(k=10, alpha=1e-4, beta=1e-2, delta=1e-2, seed=0, outer_steps=6, grid_i=4,
                grid_j=4)
    rec("cmf_dense64", bm.train_sequential, d64, bm.TrainConfig(**base), keep=True)
    rec("cmf_dense64_early", bm.train_sequential, d64,
        bm.TrainConfig(**dict(base, outer_steps=100)), early_stop=True)
    for wk in (1, 3, 4, 7):
        rec(f"cpmf_dense64_w{wk}", bm.train_sync_parallel, d64,
            bm.TrainConfig(**dict(base, workers=wk)), keep=wk == 3)
    tr, te = bm.split(d64, 0.2, seed=1)
    rec("cpmf_dense64_holdout_w4", bm.train_sync_parallel, tr,
        bm.TrainConfig(**dict(base, workers=4, outer_steps=3)), te)
    r, c, v = make_ml100k_standin()
    sd = bm.RatingsDataset(943, 1682, r, c, v)
    rec("cmf_c1_k30", bm.train_sequential, sd,
        bm.TrainConfig(k=30, outer_steps=5, grid_i=4, grid_j=4))
    rec("cpmf_c1_k30_w8", bm.train_sync_parallel, sd,
        bm.TrainConfig(k=30, outer_steps=5, grid_i=4, grid_j=4, workers=8))
    np.savez_compressed(os.path.join(OUT, "baseline_cases.npz"), **out)
    return meta


def io_cases():
    """Byte-exact outputs of the reference's writers (data_io.py:193-309)."""
    import io as _io

    d = bm.gen_synthetic(bm.SyntheticSpec(7, 5, 1, 5, seed=2, density=0.6))
    cfg = bm.TrainConfig(k=3, outer_steps=3, grid_i=2, grid_j=2, alpha=1e-2)
    tr, te = bm.split(d, 0.3, seed=1)
    res = bm.train_blocked(tr, cfg, te, early_stop=False, timing=False)
    buf_m, buf_t, buf_d = _io.StringIO(), _io.StringIO(), _io.StringIO()
    bm.save_model(res.model, buf_m)
    bm.write_trace(res.trace, buf_t, config={"k": 3, "grid": "2x2", "schedule": "const:1"})
    bm.save_dataset(d, buf_d)
    return dict(model=buf_m.getvalue(), trace=buf_t.getvalue(), dataset=buf_d.getvalue(),
                rows=d.rows.tolist(), cols=d.cols.tolist(), values=d.values.tolist(),
                u=res.model.u.tolist(), v=res.model.v.tolist(),
                train=[s.train_rmse for s in res.trace], test=[s.test_rmse for s in res.trace])


def main():
    kernel_cases()
    meta = dict(
        reference="blockmf " + bm.__version__ + " (/root/reference/pkg/src)",
        partition=partition_cases(),
        plans=plans(),
        traces=traces(),
        io=io_cases(),
        baselines=baseline_cases(),
        hand=dict(
            rmse_hand=bm.rmse(bm.FactorModel(np.array([[1.0], [2.0]]), np.array([[1.0], [2.0]])),
                              bm.RatingsDataset.from_triples(2, 2, [(0, 0, 4.0), (1, 1, 8.0)])),
            split_bounds_10_3=bm.split_bounds(10, 3).tolist(),
            locate=list(bm.locate(bm.make_grid(1024, 1024, 32, 32), 100, 200)),
        ),
    )
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
