"""The ordered stratum kernel (csrc/ordered.cu) applies every U-row and V-row
update in the reference's stored order (_kernels.py:42-55), so its factors must
equal a sequential fp32 walk with the same arithmetic (oracle/emu32.c) BIT FOR
BIT, for any slab / stage split, any k and any grid; and a step must be
bit-reproducible run to run."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _data(n, m, nnz, seed, dup=0.0):
    g = np.random.default_rng(seed)
    cells = g.choice(n * m, size=nnz, replace=False)
    r, c = cells // m, cells % m
    if dup > 0:
        k_ = int(dup * nnz)
        src, dst = g.integers(0, nnz, k_), g.integers(0, nnz, k_)
        r[dst], c[dst] = r[src], c[src]
    v = np.clip(np.rint(3.5 + g.normal(0, 1, nnz)), 1, 5)
    return r, c, v


def _padded(a, kp):
    out = np.zeros((a.shape[0], kp), np.float32)
    out[:, : a.shape[1]] = a.astype(np.float32)
    return out


def _run(n, m, nnz, I, J, k, iters, steps, stage_ratings, seed, dup=0.0, alpha=1e-3,
         beta=1e-2, warp=1):
    r, c, v = _data(n, m, nnz, seed, dup)
    eng = bm.Engine(bm.EngineOptions(ordered=True))
    eng._opt("ord_stage_ratings", float(stage_ratings))
    eng._opt("ord_warp", float(warp))
    eng.partition(r, c, v, n, m, I, J)
    eng.init_factors(n, m, k, seed)
    u0, v0 = eng.get_factors()
    kp = (k + 3) // 4 * 4
    U, V = _padded(u0, kp), _padded(v0, kp)
    off, order, lr, lc = eng.export_partition()
    x32 = v[order].astype(np.float32)
    rb, cb = np.asarray(bm.split_bounds(n, I)), np.asarray(bm.split_bounds(m, J))
    for s in range(steps):
        plan = bm.plan_step(I, J, s)
        ids, boff = eng.plan_arrays(plan)
        sse, bad = eng.run_step(ids, boff, iters, alpha, beta)
        assert bad is None
        want_sse, ebad = O.emu32_step(lr, lc, x32, off, rb, cb, J, ids, U, V, alpha, beta, iters,
                                       warp=bool(warp))
        assert ebad < 0
        np.testing.assert_allclose(sse, want_sse, rtol=1e-12, atol=1e-300)
    gu, gv = eng.get_factors()
    eng.close()
    assert np.array_equal(gu.astype(np.float32), U[:, :k]), np.abs(gu - U[:, :k]).max()
    assert np.array_equal(gv.astype(np.float32), V[:, :k]), np.abs(gv - V[:, :k]).max()
    return sse


@pytest.mark.parametrize("warp", [1, 0])
@pytest.mark.parametrize("k", [1, 3, 8, 30, 32, 64, 96, 128, 200])
def test_ordered_bit_identical_to_sequential_fp32(k, warp):
    _run(700, 500, 30_000, 3, 3, k, iters=1, steps=2, stage_ratings=1500, seed=k, warp=warp)


@pytest.mark.parametrize("I,J", [(1, 1), (4, 1), (1, 4), (3, 5), (5, 2)])
def test_ordered_grids_and_stage_splits(I, J):
    for sr in (10**9, 700, 97):  # one stage per block ... many slabs per block
        _run(400, 300, 20_000, I, J, 16, iters=2, steps=2, stage_ratings=sr, seed=I * 7 + J)


def test_ordered_dense_with_duplicates():
    """Dense rows sharing their column order (the worst case for column waits)
    and duplicate cells (two updates of one (u, v) pair in a row)."""
    _run(64, 64, 64 * 64, 1, 1, 8, iters=3, steps=2, stage_ratings=300, seed=3, dup=0.05)
    _run(200, 150, 25_000, 2, 2, 32, iters=1, steps=3, stage_ratings=2000, seed=4, dup=0.2)


def test_ordered_step_is_deterministic():
    n, m, nnz, P, k = 3000, 2000, 200_000, 4, 64
    r, c, v = _data(n, m, nnz, 11)
    outs = []
    for _ in range(2):
        eng = bm.Engine(bm.EngineOptions(ordered=True))
        eng._opt("ord_stage_ratings", 4000.0)
        eng.partition(r, c, v, n, m, P, P)
        eng.init_factors(n, m, k, 0)
        ids, off = eng.plan_arrays(bm.plan_step(P, P, 0))
        sse, _ = eng.run_step(ids, off, 2, 1e-3, 1e-2)
        u, vv = eng.get_factors()
        eng.close()
        outs.append((sse, u, vv))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][2], outs[1][2])


@pytest.mark.parametrize("I,J,stage_ratings", [(1, 1, 10**9), (2, 2, 10**9), (2, 1, 900)])
def test_ordered_converge_on_device_matches_sequential(I, J, stage_ratings):
    """ConvergeEachBlock runs its whole per-block loop inside the ordered
    kernel (sgd_converge, _kernels.py:62-100): sweep counts, capped flags and
    factors equal the sequential fp32 walk driven by the same stopping rule."""
    n, m, nnz, k, tol, cap = 500, 400, 40_000, 16, 0.002, 40
    r, c, v = _data(n, m, nnz, 21)
    eng = bm.Engine(bm.EngineOptions(ordered=True))
    eng._opt("ord_stage_ratings", float(stage_ratings))
    eng.partition(r, c, v, n, m, I, J)
    eng.init_factors(n, m, k, 0)
    u0, v0 = eng.get_factors()
    kp = (k + 3) // 4 * 4
    U, V = _padded(u0, kp), _padded(v0, kp)
    off, order, lr, lc = eng.export_partition()
    x32 = v[order].astype(np.float32)
    rb, cb = np.asarray(bm.split_bounds(n, I)), np.asarray(bm.split_bounds(m, J))
    alpha, beta = 2e-3, 1e-2
    plan = bm.plan_step(I, J, 0)
    ids, boff = eng.plan_arrays(plan)
    sse, iters_used, capped, bad = eng.run_step_converge(ids, boff, tol, cap, alpha, beta)
    assert bad is None
    for b in ids:
        cnt = off[b + 1] - off[b]
        one = np.array([b], np.int32)
        s0, _ = O.emu32_step(lr, lc, x32, off, rb, cb, J, one, U, V, alpha, beta, 0)
        prev, used, cp = np.sqrt(s0[b] / cnt), 0, True
        while used < cap:
            s1, _ = O.emu32_step(lr, lc, x32, off, rb, cb, J, one, U, V, alpha, beta, 1)
            used += 1
            now = np.sqrt(s1[b] / cnt)
            if prev - now < tol:
                cp = False
                break
            prev = now
        assert iters_used[b] == used and bool(capped[b]) == cp, (b, iters_used[b], used)
        np.testing.assert_allclose(sse[b], s1[b], rtol=1e-12)
    gu, gv = eng.get_factors()
    eng.close()
    assert np.array_equal(gu.astype(np.float32), U[:, :k])
    assert np.array_equal(gv.astype(np.float32), V[:, :k])


@pytest.mark.parametrize("I,J,stage_ratings,iters", [(1, 1, 10**9, 1), (3, 3, 700, 2),
                                                     (2, 4, 300, 1), (4, 1, 10**9, 3)])
def test_exact_ordered_bit_identical_to_reference(I, J, stage_ratings, iters):
    """Exact mode runs the ordered schedule in fp64 with the reference's own
    operation order (ordered_exact_kernel): factors and per-block SSEs equal the
    oracle's restatement of the reference (pinned to the reference's golden
    vectors) bit for bit, for any number of slabs per block."""
    n, m, nnz, k = 400, 300, 12_000, 12
    r, c, v = _data(n, m, nnz, 5, dup=0.05)
    eng = bm.Engine(bm.EngineOptions(exact=True))
    eng._opt("ord_stage_ratings", float(stage_ratings))
    eng.partition(r, c, v, n, m, I, J)
    u0, v0 = O.init_factors(n, m, k, 1)
    eng.set_factors(u0, v0)
    P = O.partition(r, c, v, n, m, I, J)
    ou, ov = u0.copy(), v0.copy()
    for s in range(3):
        ids, off = eng.plan_arrays(bm.plan_step(I, J, s))
        sse, bad = eng.run_step(ids, off, iters, 1e-3, 1e-2)
        assert bad is None
        osse, _, pos, _, _ = O.run_step(P, ou, ov, s, iters, 1e-3, 1e-2)
        assert pos < 0
        assert np.array_equal(sse, osse), np.abs(sse - osse).max()
    gu, gv = eng.get_factors()
    eng.close()
    assert np.array_equal(gu, ou) and np.array_equal(gv, ov)
