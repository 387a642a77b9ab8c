"""Post-sweep SSE kernels (the trace's per-block SSE, reference
_kernels.py:16-28 consumed at trainer.py:149-158).  The last stratum of a step
is not touched again in that step, so its blocks' SSEs must equal the SSE of
the downloaded final factors, computed here in fp64 with numpy."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm

pytestmark = pytest.mark.gpu


def _data(n, m, nnz, seed):
    g = np.random.default_rng(seed)
    cells = g.choice(n * m, size=nnz, replace=False)
    vals = np.clip(np.rint(3.5 + g.normal(0, 1, nnz)), 1, 5)
    return cells // m, cells % m, vals


@pytest.mark.parametrize("k", [8, 30, 64, 128])
def test_last_stratum_sse_matches_final_factors(k):
    n, m, nnz, P = 1500, 1100, 120_000, 4
    r, c, v = _data(n, m, nnz, seed=k)
    eng = bm.Engine()
    eng.partition(r, c, v, n, m, P, P)
    eng.init_factors(n, m, k, 0)
    plan = bm.plan_step(P, P, 0)
    ids, off = eng.plan_arrays(plan)
    for _ in range(2):
        sse, bad = eng.run_step(ids, off, 1, 1e-3, 1e-2)
        assert bad is None
    u, vv = eng.get_factors()
    rb = np.asarray(bm.split_bounds(n, P))
    cb = np.asarray(bm.split_bounds(m, P))
    bi = np.searchsorted(rb, r, side="right") - 1
    bj = np.searchsorted(cb, c, side="right") - 1
    pred = np.einsum("ij,ij->i", u[r], vv[c])
    err2 = (v - pred) ** 2
    for bi_, bj_ in plan.batches[-1].blocks:
        sel = (bi == bi_) & (bj == bj_)
        want = err2[sel].sum()
        assert abs(sse[bi_ * P + bj_] - want) <= 1e-5 * want, (bi_, bj_)
    # the other blocks are finite and positive
    assert np.all(np.isfinite(sse)) and np.all(sse > 0)


def test_sse_covers_every_entry_once():
    """alpha = 0 leaves the factors unchanged, so every block's post-sweep SSE
    must equal the SSE of the initial factors over exactly its entries."""
    n, m, nnz, P = 300, 200, 20_000, 2
    r, c, v = _data(n, m, nnz, seed=5)
    eng = bm.Engine()
    eng.partition(r, c, v, n, m, P, P)
    eng.init_factors(n, m, 128, 1)
    plan = bm.plan_step(P, P, 0)
    ids, off = eng.plan_arrays(plan)
    sse, _ = eng.run_step(ids, off, 1, 0.0, 0.0)
    u, vv = eng.get_factors()
    pred = np.einsum("ij,ij->i", u[r], vv[c])
    rb = np.asarray(bm.split_bounds(n, P))
    cb = np.asarray(bm.split_bounds(m, P))
    blk = (np.searchsorted(rb, r, side="right") - 1) * P + np.searchsorted(cb, c, side="right") - 1
    want = np.bincount(blk, weights=(v - pred) ** 2, minlength=P * P)
    np.testing.assert_allclose(sse, want, rtol=1e-5)
