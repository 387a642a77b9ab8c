"""Every kernel shape instance against the oracle: latent widths that hit the
masked and unmasked (L, V4) variants, 1-row/1-column slabs, wide/tall grids,
empty blocks, inner iterations > 1.  Fast mode within 1e-3 per epoch; exact
mode bit-identical."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _data(n, m, nnz, seed=0):
    g = np.random.default_rng(seed)
    cells = g.choice(n * m, size=nnz, replace=False)
    vals = np.clip(np.rint(3.5 + g.normal(0, 1, nnz)), 1, 5)
    return bm.RatingsDataset(n, m, cells // m, cells % m, vals)


def _compare(d, cfg, options=None, tol=1e-3):
    res = bm.train_blocked(d, cfg, early_stop=False, timing=False, options=options)
    u, v, tr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=cfg.k, alpha=cfg.alpha,
                                  beta=cfg.beta, outer_steps=cfg.outer_steps,
                                  schedule=bm.format_schedule(cfg.inner_schedule),
                                  grid_i=cfg.grid_i, grid_j=cfg.grid_j, seed=cfg.seed,
                                  early_stop=False, nthreads=8)
    got = np.array([s.train_rmse for s in res.trace])
    ref = np.array([s["train_rmse"] for s in tr])
    if options is not None and options.exact:
        assert got.tolist() == ref.tolist()
        assert np.array_equal(res.model.u, u) and np.array_equal(res.model.v, v)
    else:
        assert np.abs(got - ref).max() <= tol, (got, ref)
        assert np.abs(res.model.u - u).max() < 1e-2


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8, 10, 16, 17, 24, 30, 32, 33, 48, 64, 65, 96,
                               100, 128, 129, 192, 200, 256, 300, 384, 512])
def test_latent_widths(k):
    d = _data(700, 500, 40_000, seed=k)
    _compare(d, bm.TrainConfig(k=k, outer_steps=3, grid_i=4, grid_j=4, alpha=2e-4))


@pytest.mark.parametrize("gi,gj", [(1, 1), (3, 7), (7, 3), (16, 16), (1, 9), (40, 40)])
def test_grids(gi, gj):
    d = _data(400, 300, 30_000, seed=gi * 100 + gj)
    _compare(d, bm.TrainConfig(k=16, outer_steps=3, grid_i=gi, grid_j=gj))


def test_one_index_slabs_and_empty_blocks():
    d = _data(12, 9, 40, seed=3)  # 12x9 grid of 1x1 slabs: most blocks empty
    _compare(d, bm.TrainConfig(k=6, outer_steps=4, grid_i=12, grid_j=9, alpha=1e-2))
    _compare(d, bm.TrainConfig(k=6, outer_steps=4, grid_i=12, grid_j=9, alpha=1e-2),
             options=bm.EngineOptions(exact=True))


@pytest.mark.parametrize("g", [2, 5])
def test_inner_iterations(g):
    d = _data(900, 600, 60_000, seed=g)
    _compare(d, bm.TrainConfig(k=24, outer_steps=3, grid_i=6, grid_j=6,
                               inner_schedule=bm.Constant(g)))


def test_exact_mode_odd_shapes():
    d = _data(97, 41, 1500, seed=9)
    _compare(d, bm.TrainConfig(k=7, outer_steps=3, grid_i=5, grid_j=3, alpha=1e-3),
             options=bm.EngineOptions(exact=True))


def test_fused_and_unfused_agree():
    d = _data(2000, 1500, 150_000, seed=4)
    cfg = bm.TrainConfig(k=32, outer_steps=3, grid_i=8, grid_j=8)
    for fused in (True, False):
        _compare(d, cfg, options=bm.EngineOptions(fused=fused))
    _compare(d, cfg, options=bm.EngineOptions(bulk_red=True))
    _compare(d, cfg, options=bm.EngineOptions(sse_wide=True))
