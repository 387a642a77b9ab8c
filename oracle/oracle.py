"""CPU oracle for the BGMF hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg / ``--impl reference`` arm may import this module, and
only as the checker (or as the timed CPU reference).  The product package
``paper_2304_13724_b200`` never imports it.

It restates the reference algorithm (paths relative to
``/root/reference/pkg/src/blockmf/``):

* numeric loops: ``bgmf_oracle.c`` (``_kernels.py:16-100``), bit-identical fp64;
* ``split_bounds``            <- ``partition.py:18-37``
* ``partition``               <- ``partition.py:112-136`` (C, ``oracle_partition``)
* ``plan_step``               <- ``scheduler.py:45-75``
* ``init_factors``            <- ``core.py:179-193`` (same numpy PCG64 calls)
* ``resolve_inner_iters``     <- ``trainer.py:52-73``
* ``rmse`` / ``holdout_rmse`` <- ``metrics.py:39-81`` (same numpy reductions)
* ``train_blocked``           <- ``trainer.py:76-184``

Parity of this restatement is pinned against the reference itself by
``tests/golden/*.npz`` (made by ``tests/golden/make_golden.py``, which imports
the reference package in the build container) and ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    """Compile the C restatement (gcc, no reference sources involved)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_block_sse.restype = ctypes.c_double
        L.oracle_block_sse.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64,
                                       _f64p, _f64p, ctypes.c_int]
        L.oracle_sgd_sweeps.restype = None
        L.oracle_sgd_sweeps.argtypes = [
            _i64p, _i64p, _f64p, ctypes.c_int64, _f64p, _f64p, ctypes.c_int,
            ctypes.c_double, ctypes.c_double, ctypes.c_int,
            _f64p, _f64p, _i64p, _i64p]
        L.oracle_sgd_converge.restype = None
        L.oracle_sgd_converge.argtypes = [
            _i64p, _i64p, _f64p, ctypes.c_int64, _f64p, _f64p, ctypes.c_int,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
            _f64p, _f64p, _i64p, ctypes.POINTER(ctypes.c_int), _i64p, _i64p]
        L.oracle_gradient_steps.restype = None
        L.oracle_gradient_steps.argtypes = [
            _i64p, _i64p, _f64p, ctypes.c_int64, _f64p, ctypes.c_int64, _f64p, ctypes.c_int64,
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
            _f64p, _f64p, _i64p, _i64p]
        L.oracle_partition.restype = ctypes.c_int
        L.oracle_partition.argtypes = [
            _i64p, _i64p, _f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int, ctypes.c_int, _i64p, _i64p, _i64p, _f64p]
        L.oracle_run_step.restype = ctypes.c_int64
        L.oracle_run_step.argtypes = [
            _i64p, _i64p, _i64p, _f64p, _i64p, _i64p, ctypes.c_int, ctypes.c_int,
            _f64p, _f64p, ctypes.c_int, _i32p, _i32p, ctypes.c_int, ctypes.c_int,
            ctypes.c_double, ctypes.c_double, ctypes.c_int, _f64p, _i64p]
        L.emu32_step.restype = ctypes.c_int64
        L.emu32_step.argtypes = [
            _i32p, _i32p, ctypes.POINTER(ctypes.c_float), _i64p, _i64p, _i64p, ctypes.c_int,
            _i32p, ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_float,
            ctypes.c_int, _f64p]
        _lib = L
    return _lib


def gpu_shape(kp: int, warp: bool = False) -> tuple[int, int]:
    """Lane geometry (L, V4) of the GPU fast path for a padded row of kp floats
    (restates shape_for in paper_2304_13724_b200/csrc/rows.cuh, and with
    warp=True ordered_shape in csrc/ordered.cu; test use)."""
    f4 = kp // 4
    if warp:
        return 32, max(1, -(-f4 // 32))
    if f4 >= 6 and f4 % 3 == 0 and ((f4 // 3) & (f4 // 3 - 1)) == 0 and f4 // 3 <= 32:
        return f4 // 3, 3
    if f4 <= 2:
        return max(f4, 1), 1
    L = 4
    while L * 4 < f4 and L < 32:
        L <<= 1
    v4 = 1
    while v4 * L < f4:
        v4 <<= 1
    return L, v4


def emu32_step(lrow, lcol, val32, offsets, row_bounds, col_bounds, J, plan_ids, U32, V32,
               alpha, beta, iters, warp=True):
    """Sequential fp32 sweep in stored order with the GPU's operation shapes
    (emu32.c).  U32 / V32 (n x kp, m x kp float32) are updated in place;
    returns (per-block post-sweep SSE, first diverged plan position or -1)."""
    L = lib()
    kp = U32.shape[1]
    lv, v4 = gpu_shape(kp, warp)
    lr = np.ascontiguousarray(lrow, np.int32)
    lc = np.ascontiguousarray(lcol, np.int32)
    x = np.ascontiguousarray(val32, np.float32)
    off = np.ascontiguousarray(offsets, np.int64)
    rb = np.ascontiguousarray(row_bounds, np.int64)
    cb = np.ascontiguousarray(col_bounds, np.int64)
    pl = np.ascontiguousarray(plan_ids, np.int32)
    sse = np.zeros(len(off) - 1, np.float64)
    fp = ctypes.POINTER(ctypes.c_float)
    bad = L.emu32_step(_p(lr, _i32p), _p(lc, _i32p), _p(x, fp), _p(off, _i64p), _p(rb, _i64p),
                       _p(cb, _i64p), J, _p(pl, _i32p), len(pl), _p(U32, fp), _p(V32, fp), kp,
                       lv, v4, float(alpha), float(beta), int(iters), _p(sse, _f64p))
    return sse, int(bad)


def _p(a, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# host-side restatements


def split_bounds(n: int, parts: int) -> np.ndarray:
    """partition.py:18-37: first n % parts slabs one longer."""
    if parts < 1 or parts > n:
        raise ValueError("bad split")
    q, r = divmod(n, parts)
    sizes = np.array([q + (1 if p < r else 0) for p in range(parts)], dtype=np.int64)
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def plan_step(I: int, J: int, step: int) -> list[list[tuple[int, int]]]:
    """scheduler.py:45-75: wave t gives column j row (j+step+t) mod I; waves
    with repeated rows (J > I) split first-fit by ascending column."""
    out: list[list[tuple[int, int]]] = []
    for t in range(I):
        wave = [((j + step + t) % I, j) for j in range(J)]
        if J <= I:
            out.append(wave)
            continue
        subs: list[list[tuple[int, int]]] = []
        for blk in wave:
            for s in subs:
                if all(blk[0] != o[0] for o in s):
                    s.append(blk)
                    break
            else:
                subs.append([blk])
        out.extend(subs)
    return out


def init_factors(n: int, m: int, k: int, seed: int):
    """core.py:179-193: PCG64(seed); u drawn before v; scale 1/sqrt(k)."""
    g = np.random.default_rng(seed)
    s = 1.0 / math.sqrt(k)
    u = g.random((n, k)) * s
    v = g.random((m, k)) * s
    return u, v


def resolve_inner_iters(spec: str, step: int, ratio: float = 1.0):
    """trainer.py:52-73 for schedule strings const:G | inc:P,C | dec:S |
    adaptive:S | converge:TOL (core.py:258-292 grammar)."""
    kind, _, args = spec.partition(":")
    if kind == "const":
        return int(args)
    if kind == "inc":
        p, c = (int(x) for x in args.split(","))
        return min(math.ceil(step / p), c)
    if kind == "dec":
        return max(int(args) - step + 1, 1)
    if kind == "adaptive":
        return max(round(int(args) * ratio), 1)
    if kind == "converge":
        return None
    raise ValueError(spec)


# --------------------------------------------------------------------------
# numeric entry points (C)


def block_sse(rows, cols, vals, u, v) -> float:
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    return lib().oracle_block_sse(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                  len(rows), _p(u, _f64p), _p(v, _f64p), u.shape[1])


def sgd_sweeps(rows, cols, vals, u, v, alpha, beta, iters):
    """In-place on u, v (C-contiguous f64).  Returns the reference tuple
    (sse_before, sse_after, bad_entry, bad_iter)."""
    assert u.flags.c_contiguous and v.flags.c_contiguous
    assert u.dtype == np.float64 and v.dtype == np.float64
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    sb, sa = ctypes.c_double(), ctypes.c_double()
    be, bi = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_sgd_sweeps(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), len(rows),
                            _p(u, _f64p), _p(v, _f64p), u.shape[1], alpha, beta, iters,
                            ctypes.byref(sb), ctypes.byref(sa), ctypes.byref(be),
                            ctypes.byref(bi))
    return sb.value, sa.value, be.value, bi.value


def sgd_converge(rows, cols, vals, u, v, alpha, beta, tol, cap):
    """Reference tuple (sse_before, sse_after, iters_used, capped, bad_entry, bad_iter)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    sb, sa = ctypes.c_double(), ctypes.c_double()
    iu, cp = ctypes.c_int64(), ctypes.c_int()
    be, bi = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_sgd_converge(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), len(rows),
                              _p(u, _f64p), _p(v, _f64p), u.shape[1], alpha, beta, tol,
                              cap, ctypes.byref(sb), ctypes.byref(sa), ctypes.byref(iu),
                              ctypes.byref(cp), ctypes.byref(be), ctypes.byref(bi))
    return sb.value, sa.value, iu.value, cp.value, be.value, bi.value


def gradient_steps(rows, cols, vals, u, v, alpha, beta, iters):
    """_kernels.py:103-140, in place on u, v.  Reference tuple
    (sse_before, sse_after, bad_entry, bad_iter)."""
    assert u.flags.c_contiguous and v.flags.c_contiguous
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    sb, sa = ctypes.c_double(), ctypes.c_double()
    be, bi = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_gradient_steps(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), len(rows),
                                _p(u, _f64p), u.shape[0], _p(v, _f64p), v.shape[0], u.shape[1],
                                alpha, beta, iters, ctypes.byref(sb), ctypes.byref(sa),
                                ctypes.byref(be), ctypes.byref(bi))
    return sb.value, sa.value, be.value, bi.value


def block_gradients(rows, cols, vals, u, v, beta):
    """kernel.py:161-179 restated in numpy: (objective, gu, gv)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    e = np.asarray(vals, np.float64) - np.einsum("ij,ij->i", u[rows], v[cols])
    gu = beta * u
    gv = beta * v
    np.add.at(gu, rows, -2.0 * e[:, None] * v[cols])
    np.add.at(gv, cols, -2.0 * e[:, None] * u[rows])
    reg = np.square(u).sum() + np.square(v).sum()
    return float(e @ e + 0.5 * beta * reg), gu, gv


def partition(rows, cols, vals, n: int, m: int, I: int, J: int) -> dict:
    """BlockedDataset internals of partition.py:112-136."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    nnz = len(rows)
    off = np.zeros(I * J + 1, np.int64)
    lr = np.empty(nnz, np.int64)
    lc = np.empty(nnz, np.int64)
    lv = np.empty(nnz, np.float64)
    rc = lib().oracle_partition(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), nnz,
                                n, m, I, J, _p(off, _i64p), _p(lr, _i64p), _p(lc, _i64p),
                                _p(lv, _f64p))
    if rc != 0:
        raise MemoryError("oracle_partition failed")
    return dict(offsets=off, rows=lr, cols=lc, values=lv,
                row_bounds=split_bounds(n, I), col_bounds=split_bounds(m, J),
                I=I, J=J, n=n, m=m)


def flat_plan(I: int, J: int, step: int):
    batches = plan_step(I, J, step)
    ids = np.array([bi * J + bj for b in batches for bi, bj in b], np.int32)
    off = np.zeros(len(batches) + 1, np.int32)
    off[1:] = np.cumsum([len(b) for b in batches])
    return batches, ids, off


def run_step(P: dict, u, v, step0: int, iters: int, alpha: float, beta: float,
             nthreads: int = 1):
    """One outer step (0-based step0) over partition P; returns
    (sse_after[I*J], bad[I*J,2], first_bad_plan_pos, batches)."""
    I, J = P["I"], P["J"]
    batches, ids, off = flat_plan(I, J, step0)
    sse = np.zeros(I * J, np.float64)
    bad = np.full((I * J, 2), -1, np.int64)
    pos = lib().oracle_run_step(
        _p(P["offsets"], _i64p), _p(P["rows"], _i64p), _p(P["cols"], _i64p),
        _p(P["values"], _f64p), _p(P["row_bounds"], _i64p), _p(P["col_bounds"], _i64p),
        I, J, _p(u, _f64p), _p(v, _f64p), u.shape[1], _p(ids, _i32p), _p(off, _i32p),
        len(batches), iters, alpha, beta, nthreads, _p(sse, _f64p), _p(bad, _i64p))
    return sse, bad, int(pos), batches, ids


def predict(u, v, rows, cols, chunk: int = 1 << 20) -> np.ndarray:
    """core.py:163-165 (einsum over gathered rows), evaluated in row chunks:
    each prediction is the same per-row dot, but the gathers stay at chunk x k
    instead of materialising nnz x k fp64 twice (2 x 102 GB at C4)."""
    out = np.empty(len(rows), np.float64)
    for s in range(0, len(rows), chunk):
        e = min(len(rows), s + chunk)
        out[s:e] = np.einsum("ij,ij->i", u[rows[s:e]], v[cols[s:e]])
    return out


def rmse(u, v, rows, cols, vals) -> float:
    """metrics.py:39-52 (predictions, then numpy's pairwise sum over the whole
    squared-error vector)."""
    err = vals - predict(u, v, rows, cols)
    return float(np.sqrt(np.sum(np.square(err)) / len(vals)))


def holdout_rmse(u, v, train_rows, train_cols, train_vals, test_rows, test_cols,
                 test_vals) -> float:
    """metrics.py:55-81: cold entries (row or col unseen in train) predict the
    train mean."""
    n, m = u.shape[0], v.shape[0]
    rs = np.zeros(n, bool)
    cs = np.zeros(m, bool)
    rs[train_rows] = True
    cs[train_cols] = True
    cold = ~(rs[test_rows] & cs[test_cols])
    fb = float(train_vals.mean()) if len(train_vals) else 0.0
    pred = predict(u, v, test_rows, test_cols)
    pred[cold] = fb
    err = test_vals - pred
    return float(np.sqrt(np.sum(np.square(err)) / len(test_vals)))


class OracleDivergence(RuntimeError):
    def __init__(self, block, entry, iteration, step, trace):
        super().__init__(f"block {block}: non-finite residual at entry {entry}, "
                         f"inner iteration {iteration}; reduce alpha")
        self.block, self.entry, self.iteration, self.step = block, entry, iteration, step
        self.partial_trace = trace


def train_blocked(n, m, rows, cols, vals, *, k=10, alpha=1e-4, beta=1e-2, delta=1e-2,
                  outer_steps=100, schedule="const:1", grid_i=1, grid_j=1, seed=0,
                  test=None, early_stop=True, nthreads=1, converge_cap=10_000,
                  P=None):
    """trainer.py:76-184.  ``test`` is (rows, cols, vals) or None.  Returns
    (u, v, trace, stop_reason); trace is a list of dicts with the TraceStep
    fields (seconds measured with perf_counter)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    if P is None:
        P = partition(rows, cols, vals, n, m, grid_i, grid_j)
    u, v = init_factors(n, m, k, seed)
    adaptive = schedule.startswith("adaptive")
    converge = schedule.startswith("converge")
    tol = float(schedule.partition(":")[2]) if converge else 0.0
    hist = [rmse(u, v, rows, cols, vals)] if adaptive and len(rows) else [0.0]
    trace: list[dict] = []
    stop = "max_steps"
    for step in range(1, outer_steps + 1):
        if adaptive and step >= 2:
            prev, cur = hist[-2], hist[-1]
            ratio = (prev - cur) / prev if prev > 0 else 0.0
        else:
            ratio = 1.0
        g = resolve_inner_iters(schedule, step, ratio)
        t0 = time.perf_counter()
        sse_tot, cnt_tot, max_it, capped = 0.0, 0, 0, 0
        if g is not None:
            sse, bad, pos, batches, ids = run_step(P, u, v, step - 1, g, alpha, beta,
                                                   nthreads)
            if pos >= 0:
                b = int(ids[pos])
                raise OracleDivergence((b // grid_j, b % grid_j), int(bad[b, 0]),
                                       int(bad[b, 1]), step, trace)
            for b in ids:  # merge in submission order (trainer.py:149-152)
                sse_tot = sse_tot + float(sse[b])
                cnt_tot += int(P["offsets"][b + 1] - P["offsets"][b])
            max_it = g
        else:
            for batch in plan_step(grid_i, grid_j, step - 1):
                for bi, bj in batch:
                    b = bi * grid_j + bj
                    lo, hi = P["offsets"][b], P["offsets"][b + 1]
                    r0, r1 = P["row_bounds"][bi], P["row_bounds"][bi + 1]
                    c0, c1 = P["col_bounds"][bj], P["col_bounds"][bj + 1]
                    us, vs = u[r0:r1], v[c0:c1]
                    _, sa, it, cp, be, bit = sgd_converge(
                        P["rows"][lo:hi], P["cols"][lo:hi], P["values"][lo:hi], us, vs,
                        alpha, beta, tol, converge_cap)
                    if be >= 0:
                        raise OracleDivergence((bi, bj), be, bit, step, trace)
                    sse_tot = sse_tot + sa
                    cnt_tot += int(hi - lo)
                    max_it = max(max_it, it)
                    capped += cp
        train = 0.0 if cnt_tot == 0 else float(np.sqrt(sse_tot / cnt_tot))
        test_rmse = None
        if test is not None and len(test[0]) > 0:
            test_rmse = holdout_rmse(u, v, rows, cols, vals, *test)
        trace.append(dict(step=step, train_rmse=train, test_rmse=test_rmse,
                          seconds=time.perf_counter() - t0, inner_iters=max_it,
                          capped_blocks=capped))
        hist.append(train)
        if early_stop:
            if cnt_tot == 0:
                stop = "converged"
                break
            if len(trace) >= 2 and trace[-2]["train_rmse"] - train < delta:
                stop = "converged"
                break
    return u, v, trace, stop


def train_sync_parallel(n, m, rows, cols, vals, *, k=10, alpha=1e-4, beta=1e-2, delta=1e-2,
                        outer_steps=100, seed=0, workers=1, test=None, early_stop=True):
    """baselines.py:100-182 (CPMF): row shards over the row-major 1x1
    partition, each swept once per step on the shared U and a private copy
    of V, V deltas summed in shard order.  Returns (u, v, trace, stop)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    P = partition(rows, cols, vals, n, m, 1, 1)
    wr, wc, wv = P["rows"], P["cols"], P["values"]
    u, v = init_factors(n, m, k, seed)
    shards = min(workers, max(n, 1))
    edges = np.searchsorted(wr, split_bounds(n, shards))
    trace: list[dict] = []
    stop = "max_steps"
    for step in range(1, outer_steps + 1):
        t0 = time.perf_counter()
        results = []
        if shards == 1:
            out = sgd_sweeps(wr, wc, wv, u, v, alpha, beta, 1)
            results.append((out, int(edges[1] - edges[0])))
        else:
            v_start = v.copy()
            privates = [v_start.copy() for _ in range(shards)]
            for w in range(shards):
                lo, hi = edges[w], edges[w + 1]
                out = sgd_sweeps(wr[lo:hi], wc[lo:hi], wv[lo:hi], u, privates[w], alpha, beta, 1)
                results.append((out, int(hi - lo)))
            delta_v = np.zeros_like(v)
            for v_w in privates:
                delta_v += v_w - v_start
            v[:] = v_start + delta_v
        for w, (out, _) in enumerate(results):
            if out[2] >= 0:
                raise OracleDivergence(None, int(out[2]), int(out[3]), step, trace)
        sse = sum(r[0][1] for r in results)
        count = sum(r[1] for r in results)
        test_rmse = None
        if test is not None:
            test_rmse = holdout_rmse(u, v, rows, cols, vals, *test)
        trace.append(dict(step=step, train_rmse=float(np.sqrt(sse / count)) if count else 0.0,
                          test_rmse=test_rmse, seconds=time.perf_counter() - t0,
                          inner_iters=1, capped_blocks=0))
        if early_stop:
            if count == 0 or (len(trace) >= 2 and
                              trace[-2]["train_rmse"] - trace[-1]["train_rmse"] < delta):
                stop = "converged"
                break
    return u, v, trace, stop
