"""End-to-end training on the GPU against the reference.

* exact mode (fp64 sequential-per-block kernels): bit-identical traces and
  factors to the reference golden runs;
* fast mode (fp32 lossless warp-per-rating kernels, the throughput path):
  per-epoch train/test RMSE within 1e-3 absolute of the reference/oracle
  (BASELINE.md tolerance), on C1 (golden) and C2/C3 (oracle, same inputs).
"""

import math

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from helpers import config_of, sha, trace_inputs
from oracle import oracle as O
from paper_2304_13724_b200 import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-3  # absolute, per epoch (BASELINE.md "RMSE parity")
EXACT = bm.EngineOptions(exact=True)

TRACES = ["dense64_const1", "dense64_const3", "dense64_dec4", "dense64_inc", "dense64_adaptive",
          "dense64_converge", "dense64_early", "dense64_wide_2x5", "dense64_tall_5x2",
          "dense64_holdout", "c1_k30", "c1_k10", "c1_split"]


@pytest.mark.parametrize("name", TRACES)
def test_exact_mode_bit_identical(golden, name):
    meta = golden["traces"][name]
    d, te = trace_inputs(name)
    res = bm.train_blocked(d, config_of(meta), te, early_stop=meta["early_stop"], timing=False,
                           options=EXACT)
    assert [s.train_rmse for s in res.trace] == meta["train"]
    assert [s.inner_iters for s in res.trace] == meta["inner"]
    assert [s.capped_blocks for s in res.trace] == meta["capped"]
    assert res.stop_reason == meta["stop"]
    assert sha(res.model.u) == meta["u_sha"] and sha(res.model.v) == meta["v_sha"]
    if meta["test"][0] is not None:  # GPU reduction order vs numpy pairwise sum
        for a, b in zip([s.test_rmse for s in res.trace], meta["test"]):
            assert a == pytest.approx(b, rel=1e-12)
    assert bm.rmse(res.model, d) == pytest.approx(meta["final_rmse"], rel=1e-12)


@pytest.mark.parametrize("name", TRACES)
def test_fast_mode_within_tolerance(golden, name):
    meta = golden["traces"][name]
    d, te = trace_inputs(name)
    res = bm.train_blocked(d, config_of(meta), te, early_stop=meta["early_stop"], timing=False)
    got = [s.train_rmse for s in res.trace]
    assert len(got) == len(meta["train"])
    assert np.max(np.abs(np.array(got) - np.array(meta["train"]))) <= TOL
    if meta["test"][0] is not None:
        got_t = np.array([s.test_rmse for s in res.trace])
        assert np.max(np.abs(got_t - np.array(meta["test"]))) <= TOL
    assert abs(bm.rmse(res.model, d) - meta["final_rmse"]) <= TOL
    if not name.endswith("converge"):
        assert [s.inner_iters for s in res.trace] == meta["inner"]


def test_c1_parity_per_epoch_detail(golden):
    """C1 (north-star parity config): 20 epochs, k=30, 4x4 -- report the drift."""
    meta = golden["traces"]["c1_k30"]
    d, _ = trace_inputs("c1_k30")
    res = bm.train_blocked(d, config_of(meta), early_stop=False, timing=False)
    drift = np.abs(np.array([s.train_rmse for s in res.trace]) - np.array(meta["train"]))
    print("C1 max |d train_rmse| over 20 epochs:", drift.max())
    assert drift.max() <= TOL
    assert np.all(np.diff([s.train_rmse for s in res.trace]) < 0)


def _oracle_vs_gpu(name, epochs, nnz=None, k=None, grid=None):
    w = workloads.CONFIGS[name]
    k = k or w.k
    grid = grid or w.grid
    r, c, v = workloads.lowrank(w.n, w.m, nnz or w.nnz, seed=0)
    d = bm.RatingsDataset(w.n, w.m, r, c, v)
    tr, te = bm.split(d, 0.2, seed=0)
    cfg = bm.TrainConfig(k=k, alpha=w.alpha, beta=w.beta, outer_steps=epochs, grid_i=grid,
                         grid_j=grid, seed=0)
    res = bm.train_blocked(tr, cfg, te, early_stop=False, timing=False)
    _, _, otr, _ = O.train_blocked(tr.n, tr.m, tr.rows, tr.cols, tr.values, k=k, alpha=w.alpha,
                                   beta=w.beta, outer_steps=epochs, grid_i=grid, grid_j=grid,
                                   seed=0, test=(te.rows, te.cols, te.values), early_stop=False,
                                   nthreads=8)
    dtr = np.abs(np.array([s.train_rmse for s in res.trace]) - [s["train_rmse"] for s in otr])
    dte = np.abs(np.array([s.test_rmse for s in res.trace]) - [s["test_rmse"] for s in otr])
    print(f"{name}: max |d train| {dtr.max():.3e}  max |d test| {dte.max():.3e}")
    return dtr, dte


def test_c2_parity_vs_oracle():
    dtr, dte = _oracle_vs_gpu("C2", epochs=10)
    assert dtr.max() <= TOL and dte.max() <= TOL


@pytest.mark.slow
def test_c3_parity_vs_oracle():
    dtr, dte = _oracle_vs_gpu("C3", epochs=3)
    assert dtr.max() <= TOL and dte.max() <= TOL


class TestReferenceTrainerBehaviour:
    def cfg64(self, **kw):
        base = dict(k=10, alpha=1e-4, beta=1e-2, delta=1e-2, seed=0, outer_steps=10,
                    inner_schedule=bm.Constant(1), grid_i=4, grid_j=4)
        base.update(kw)
        return bm.TrainConfig(**base)

    def test_early_stop_and_budget(self, dense64):
        r = bm.train_blocked(dense64, self.cfg64(delta=10.0, outer_steps=50))
        assert r.stop_reason == "converged" and len(r.trace) == 2
        r = bm.train_blocked(dense64, self.cfg64(outer_steps=7), early_stop=False)
        assert r.stop_reason == "max_steps" and [s.step for s in r.trace] == list(range(1, 8))

    def test_empty_dataset(self):
        r = bm.train_blocked(bm.RatingsDataset.from_triples(4, 4, []), self.cfg64(grid_i=2,
                                                                                 grid_j=2))
        assert r.stop_reason == "converged" and len(r.trace) == 1
        assert r.trace.last().train_rmse == 0.0

    def test_holdout_only_when_given(self, dense64):
        tr, te = bm.split(dense64, 0.2, seed=1)
        a = bm.train_blocked(tr, self.cfg64(outer_steps=2), te, early_stop=False)
        b = bm.train_blocked(tr, self.cfg64(outer_steps=2), early_stop=False)
        assert all(s.test_rmse is not None for s in a.trace)
        assert all(s.test_rmse is None for s in b.trace)

    def test_hooks_and_slice_exclusivity(self, dense64):
        events, active, violations = [], {}, []

        def hook(phase, task):
            events.append((phase, task.bi, task.bj))
            if phase == "start":
                for bi, bj in active.values():
                    if bi == task.bi or bj == task.bj:
                        violations.append(((bi, bj), (task.bi, task.bj)))
                active[id(task)] = (task.bi, task.bj)
            else:
                active.pop(id(task), None)

        bm.train_blocked(dense64, self.cfg64(outer_steps=2), early_stop=False, block_hook=hook)
        starts = [(bi, bj) for p, bi, bj in events if p == "start"]
        assert len(starts) == 32 and set(starts) == {(i, j) for i in range(4) for j in range(4)}
        assert violations == []

    def test_divergence(self, dense64):
        with pytest.raises(bm.DivergenceError) as info:
            bm.train_blocked(dense64, self.cfg64(alpha=10.0), early_stop=False)
        err = info.value
        assert err.step == 1 and err.block is not None
        assert isinstance(err.partial_trace, bm.ConvergenceTrace)
        assert "reduce alpha" in str(err)

    def test_more_inner_iterations_hurt_at_equal_budget(self, dense256):
        finals = {}
        for g in (1, 8):
            cfg = self.cfg64(grid_i=8, grid_j=8, outer_steps=400 // g,
                             inner_schedule=bm.Constant(g))
            finals[g] = bm.rmse(bm.train_blocked(dense256, cfg, early_stop=False).model, dense256)
        assert finals[1] < finals[8]

    def test_fast_repeat_runs_close(self, dense64):
        a = bm.train_blocked(dense64, self.cfg64(), early_stop=False)
        b = bm.train_blocked(dense64, self.cfg64(), early_stop=False)
        da = np.abs(np.array([s.train_rmse for s in a.trace]) - [s.train_rmse for s in b.trace])
        assert da.max() <= 1e-5

    def test_exact_repeat_runs_bit_identical(self, dense64):
        a = bm.train_blocked(dense64, self.cfg64(), early_stop=False, options=EXACT)
        b = bm.train_blocked(dense64, self.cfg64(), early_stop=False, options=EXACT)
        assert a.model == b.model


def test_metrics_on_gpu(dense32):
    model = bm.FactorModel(np.array([[1.0], [2.0]]), np.array([[1.0], [2.0]]))
    d = bm.RatingsDataset.from_triples(2, 2, [(0, 0, 4.0), (1, 1, 8.0)])
    assert bm.rmse(model, d) == pytest.approx(3.5355339059327378, rel=1e-15)
    assert bm.rmse(bm.FactorModel(np.array([[2.0]]), np.array([[3.0]])),
                   bm.RatingsDataset.from_triples(1, 1, [(0, 0, 6.0)])) == 0.0
    with pytest.raises(bm.DataError, match="empty"):
        bm.rmse(bm.init_factors(2, 2, 1, 0), bm.RatingsDataset.from_triples(2, 2, []))
    with pytest.raises(bm.DataError, match="3x3"):
        bm.rmse(bm.init_factors(3, 3, 1, 0), bm.RatingsDataset.from_triples(2, 2, [(0, 0, 1.0)]))
    train = bm.RatingsDataset.from_triples(3, 3, [(0, 0, 2.0), (1, 1, 4.0)])
    ev = bm.HoldoutEvaluator(train, bm.RatingsDataset.from_triples(3, 3, [(2, 2, 3.0)]))
    assert ev.cold_entries == 1 and ev.fallback == 3.0
    assert ev.rmse(bm.init_factors(3, 3, 2, seed=0)) == 0.0
    m = bm.init_factors(32, 32, 4, seed=1)
    ref = O.rmse(m.u, m.v, dense32.rows, dense32.cols, dense32.values)
    assert bm.rmse(m, dense32) == pytest.approx(ref, rel=1e-13)
    pred = m.predict(dense32.rows, dense32.cols)
    assert np.allclose(pred, np.einsum("ij,ij->i", m.u[dense32.rows], m.v[dense32.cols]),
                       rtol=1e-14, atol=0)
    tr, te = bm.split(dense32, 0.25, seed=3)
    assert bm.test_rmse(m, tr, te) == bm.HoldoutEvaluator(tr, te).rmse(m)
    with pytest.raises(ValueError, match="share global dimensions"):
        bm.HoldoutEvaluator(dense32, bm.RatingsDataset.from_triples(8, 8, [(0, 0, 1.0)]))
    with pytest.raises(bm.DataError, match="non-empty"):
        bm.HoldoutEvaluator(dense32, bm.RatingsDataset.from_triples(32, 32, []))


@pytest.mark.slow
def test_c4_parity_vs_oracle():
    """C4 at full size (the headline config: 100M ratings, k=128, 16x16, the
    bench's alpha/beta): 2 epochs through the public API against the oracle's
    fp64 restatement of the reference on the same input -- per-epoch train
    RMSE within 1e-3, final full-set RMSE within 1e-3, finite model; exact
    mode bit-identical (trace, U, V)."""
    w = workloads.CONFIGS["C4"]
    r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=w.seed)
    d = bm.RatingsDataset(w.n, w.m, r, c, v)
    cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, outer_steps=2, grid_i=w.grid,
                         grid_j=w.grid, seed=w.seed)
    res = bm.train_blocked(d, cfg, early_stop=False)
    tr = [s.train_rmse for s in res.trace]
    assert all(math.isfinite(x) for x in tr) and tr[1] < tr[0]
    assert np.all(np.isfinite(res.model.u)) and np.all(np.isfinite(res.model.v))
    ou, ov, otr, _ = O.train_blocked(w.n, w.m, r, c, v, k=w.k, alpha=w.alpha, beta=w.beta,
                                     outer_steps=2, grid_i=w.grid, grid_j=w.grid, seed=w.seed,
                                     early_stop=False, nthreads=16)
    drift = np.abs(np.array(tr) - [s["train_rmse"] for s in otr])
    print(f"C4 max |d train_rmse| over 2 epochs: {drift.max():.3e}")
    assert drift.max() <= TOL
    assert abs(bm.rmse(res.model, d) - O.rmse(ou, ov, d.rows, d.cols, d.values)) <= TOL
    # exact mode (fp64, the ordered schedule) at full size: bit-identical to
    # the reference epoch -- trace and both factor matrices
    ex = bm.train_blocked(d, cfg, early_stop=False, options=bm.EngineOptions(exact=True))
    assert [s.train_rmse for s in ex.trace] == [s["train_rmse"] for s in otr]
    assert np.array_equal(ex.model.u, ou) and np.array_equal(ex.model.v, ov)


@pytest.mark.slow
def test_c4_zipf_parity_vs_oracle():
    """C4Z: the C4 shape with heavy-tailed users and items (the hottest item
    rated by about half the users, heavy users rating most items): hot V rows
    take many concurrent updates and heavy users' runs span chunks.  2 epochs
    against the oracle: per-epoch train RMSE and final RMSE within 1e-3."""
    w = workloads.CONFIGS["C4Z"]
    r, c, v = workloads.generate("C4Z")
    d = bm.RatingsDataset(w.n, w.m, r, c, v)
    cfg = bm.TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, outer_steps=2, grid_i=w.grid,
                         grid_j=w.grid, seed=w.seed)
    res = bm.train_blocked(d, cfg, early_stop=False)
    tr = [s.train_rmse for s in res.trace]
    assert all(math.isfinite(x) for x in tr) and tr[1] < tr[0]
    ou, ov, otr, _ = O.train_blocked(w.n, w.m, r, c, v, k=w.k, alpha=w.alpha, beta=w.beta,
                                     outer_steps=2, grid_i=w.grid, grid_j=w.grid, seed=w.seed,
                                     early_stop=False, nthreads=16)
    drift = np.abs(np.array(tr) - [s["train_rmse"] for s in otr])
    print(f"C4Z max |d train_rmse| over 2 epochs: {drift.max():.3e}")
    assert drift.max() <= TOL
    assert abs(bm.rmse(res.model, d) - O.rmse(ou, ov, d.rows, d.cols, d.values)) <= TOL


def test_exact_run_saves_reference_bytes(golden):
    """Exact mode end to end: the saved model file is byte-identical to the
    reference's save_model output for the same run (data_io.py:221-227)."""
    import io as _io

    g = golden["io"]
    d = bm.gen_synthetic(bm.SyntheticSpec(7, 5, 1, 5, seed=2, density=0.6))
    tr, te = bm.split(d, 0.3, seed=1)
    cfg = bm.TrainConfig(k=3, outer_steps=3, grid_i=2, grid_j=2, alpha=1e-2)
    res = bm.train_blocked(tr, cfg, te, early_stop=False, timing=False, options=EXACT)
    buf = _io.StringIO()
    bm.save_model(res.model, buf)
    assert buf.getvalue() == g["model"]
    assert [s.train_rmse for s in res.trace] == g["train"]


def test_run_steps_batched_matches_per_step_loop():
    """train_blocked without early stopping enqueues every epoch in one
    bgmf_run_steps call; the trace must match the per-step loop (early_stop
    with an unreachable delta) within run-to-run fp32 noise, including a
    schedule whose inner iterations vary per step, and divergence must be
    reported at the same step / block.  (delta = 0: the per-step loop would
    only stop on a rising RMSE, which these 4 epochs never show.)"""
    r, c, v = workloads.lowrank(6040, 3706, 300_000, seed=4)
    d = bm.RatingsDataset(6040, 3706, r, c, v)
    for sched in (bm.Constant(1), bm.Decreasing(3)):
        cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8, inner_schedule=sched,
                             delta=0.0)
        a = bm.train_blocked(d, cfg, early_stop=False, timing=True)
        b = bm.train_blocked(d, cfg, early_stop=True, timing=True)
        assert [s.inner_iters for s in a.trace] == [s.inner_iters for s in b.trace]
        np.testing.assert_allclose([s.train_rmse for s in a.trace],
                                   [s.train_rmse for s in b.trace], rtol=1e-5)
        assert all(s.seconds > 0 for s in a.trace)
    cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8, alpha=1e9, delta=0.0)
    errs = []
    for es in (False, True):
        with pytest.raises(bm.DivergenceError) as ei:
            bm.train_blocked(d, cfg, early_stop=es)
        errs.append((ei.value.step, ei.value.block))
    assert errs[0] == errs[1] and errs[0][0] == 1


@pytest.mark.parametrize("sched,spec", [
    (bm.Constant(2), "const:2"), (bm.IncreasingEvery(2, 3), "inc:2,3"),
    (bm.Decreasing(3), "dec:3"), (bm.AdaptiveDecreasing(3), "adaptive:3"),
    (bm.ConvergeEachBlock(0.05), "converge:0.05")], ids=lambda x: str(x)[:12])
def test_every_schedule_with_holdout_vs_oracle(sched, spec):
    """C2-shaped data (k=32, 8x8) with an 80/20 split, fast mode, every inner
    schedule of trainer.py:52-73: per-epoch train and test RMSE within 1e-3 of
    the oracle, the same inner-iteration counts (and capped blocks for
    converge, whose per-block sweep counts can differ by one where an
    improvement sits at the tolerance)."""
    r, c, v = workloads.lowrank(6040, 3706, 300_000, seed=21)
    d, te = bm.split(bm.RatingsDataset(6040, 3706, r, c, v), 0.2, seed=2)
    cfg = bm.TrainConfig(k=32, outer_steps=5, grid_i=8, grid_j=8, inner_schedule=sched)
    res = bm.train_blocked(d, cfg, te, early_stop=False)
    _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=5,
                                   grid_i=8, grid_j=8, schedule=spec, early_stop=False,
                                   test=(te.rows, te.cols, te.values), nthreads=8)
    dtr = np.abs(np.array([s.train_rmse for s in res.trace]) - [s["train_rmse"] for s in otr])
    dte = np.abs(np.array([s.test_rmse for s in res.trace]) - [s["test_rmse"] for s in otr])
    assert dtr.max() <= TOL and dte.max() <= TOL
    got_it = [s.inner_iters for s in res.trace]
    want_it = [s["inner_iters"] for s in otr]
    if spec.startswith("converge"):
        assert all(abs(a - b) <= 1 for a, b in zip(got_it, want_it))
    else:
        assert got_it == want_it


@pytest.mark.parametrize("n,m,k", [(1, 2676, 24), (2, 2000, 32), (1, 3000, 128)])
def test_heavy_user_runs_split_across_chunks(n, m, k):
    """A user whose run spans many chunks (here: every rating of a 1-2 row
    dense matrix) is swept by several groups at once; each red.adds its u
    deltas and re-reads the row once per triple batch (every L ratings), so the run
    sees the other groups' updates.  Without the re-read the trace drifted 5%
    (randomised sweep, scripts/fuzz_parity.py).  A 1x1 grid is one block per
    batch, so the auto routing runs it through the ordered kernel (every
    update in the reference's order): within the flat 1e-3 tolerance."""
    g = np.random.default_rng(0)
    cells = g.choice(n * m, n * m, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, n * m)), 1, 5)
    d = bm.RatingsDataset(n, m, r, c, v)
    cfg = bm.TrainConfig(k=k, outer_steps=2, grid_i=1, grid_j=1, alpha=2e-4,
                         inner_schedule=bm.Constant(2))
    res = bm.train_blocked(d, cfg, early_stop=False)
    _, _, otr, _ = O.train_blocked(n, m, r, c, v, k=k, outer_steps=2, grid_i=1, grid_j=1,
                                   alpha=2e-4, schedule="const:2", early_stop=False)
    got = np.array([s.train_rmse for s in res.trace])
    want = np.array([s["train_rmse"] for s in otr])
    assert np.all(np.abs(got - want) <= 1e-3), np.abs(got - want).max()


def test_run_steps_reports_late_divergence_block():
    """bgmf_run_steps queues many steps before reading their divergence words.
    Positions are step-relative: on a 255 x 255 grid the second step starts
    past global position 65000, beyond pack_bad's 16-bit field.  One rating of
    1e36 (finite, but the next update of its cell overflows fp32) sits in block X; step 1's plan
    leaves X out, step 2 sweeps it at plan position ~1000.  The block, entry
    and iteration run_steps reports must be the ones a step-by-step run
    reports (ordered mode: deterministic)."""
    n, m, P, k = 600, 600, 255, 4
    g = np.random.default_rng(3)
    cells = g.choice(n * m, 20_000, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, len(cells))), 1, 5)
    plan1 = bm.plan_step(P, P, 1)
    rb, cb = np.asarray(bm.split_bounds(n, P)), np.asarray(bm.split_bounds(m, P))
    flat = [blk for b in plan1.batches for blk in b] if hasattr(plan1, "batches") else \
        [blk for b in plan1 for blk in b]
    bi, bj = flat[1000]
    r = np.append(r, [rb[bi], rb[bi]])  # the 1e36 rating, then a duplicate cell
    c = np.append(c, [cb[bj], cb[bj]])
    v = np.append(v, [1e36, 3.0])
    engs = []
    for _ in range(2):
        e = bm.Engine(bm.EngineOptions(ordered=True))
        e.partition(r, c, v, n + 0, m, P, P)
        e.init_factors(n, m, k, 0)
        engs.append(e)
    a, b = engs
    i1, o1 = a.plan_arrays(plan1)
    X = bi * P + bj
    keep = i1 != X
    i0 = i1[keep]  # step 1: every block of the plan but X, one batch per old batch
    o0 = np.array([np.count_nonzero(keep[:o]) for o in o1], np.int32)
    _, bad, _ = a.run_steps([(i0, o0, 1), (i1, o1, 1)], 1e-3, 1e-2)
    _, bad0 = b.run_step(i0, o0, 1, 1e-3, 1e-2)
    _, bad1 = b.run_step(i1, o1, 1, 1e-3, 1e-2)
    a.close()
    b.close()
    assert bad0 is None and bad1 is not None and bad is not None
    assert int(i1[bad1[0]]) == X and bad1[0] >= 1000
    assert bad[0] == 1 and bad[1] == X and tuple(bad[2:]) == tuple(bad1[1:]), (bad, bad1)
