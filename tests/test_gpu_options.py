"""Sweep-variant options (include/bgmf.h bgmf_set_option), each forced on for a
C2 run against the oracle: the variants that are measured and kept off
(dyn_split, snap, u_ring, fuse_sse), the routed ones forced (u_prefetch, the
ordered kernel) and spread off -- every one must stay within the flat 1e-3
per-epoch tolerance, so a variant can be switched on without a parity cost."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from oracle import oracle as O
from paper_2304_13724_b200 import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-3
EPOCHS = 3


@pytest.fixture(scope="module")
def c2():
    w = workloads.CONFIGS["C2"]
    r, c, v = workloads.generate("C2")
    d = bm.RatingsDataset(w.n, w.m, r, c, v)
    cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, outer_steps=EPOCHS,
                         grid_i=w.grid, grid_j=w.grid, seed=w.seed)
    _, _, otr, _ = O.train_blocked(w.n, w.m, r, c, v, k=w.k, alpha=w.alpha, beta=w.beta,
                                   outer_steps=EPOCHS, grid_i=w.grid, grid_j=w.grid,
                                   seed=w.seed, early_stop=False, nthreads=16)
    return d, cfg, np.array([s["train_rmse"] for s in otr])


@pytest.mark.parametrize("opts", ["dyn_split=4", "snap=64", "u_prefetch=1", "spread=0",
                                  "u_ring=1", "fuse_sse=1", "ordered=1", "pdl=0",
                                  "dyn_split=2,snap=32,u_prefetch=1"])
def test_option_within_tolerance(c2, monkeypatch, opts):
    d, cfg, want = c2
    monkeypatch.setenv("BGMF_ENGINE_OPTS", opts)
    res = bm.train_blocked(d, cfg, early_stop=False)
    got = np.array([s.train_rmse for s in res.trace])
    assert np.all(np.isfinite(got)) and got[-1] < got[0]
    assert np.abs(got - want).max() <= TOL, (opts, got, want)
