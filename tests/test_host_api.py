"""Host-side logic of the drop-in API (no GPU): schedule, grid, config,
dataset types, generators -- pinned to the reference's golden values."""

import numpy as np
import pytest
from hypothesis import given, strategies as st

import paper_2304_13724_b200 as bm
from helpers import sha
from paper_2304_13724_b200 import workloads


class TestScheduler:
    def test_all_plans_equal_reference(self, golden):
        for key, text in golden["plans"].items():
            I, J, s = map(int, key.split(","))
            assert bm.format_plan(bm.plan_step(I, J, s)) == text

    def test_3x3_and_wide(self):
        assert bm.format_plan(bm.plan_step(3, 3, 0)) == (
            "(0,0) (1,1) (2,2)\n(1,0) (2,1) (0,2)\n(2,0) (0,1) (1,2)")
        assert bm.format_plan(bm.plan_step(2, 3, 0)) == "(0,0) (1,1)\n(0,2)\n(1,0) (0,1)\n(1,2)"

    def test_exhaustive_validity(self):
        for I in range(1, 9):
            for J in range(1, 9):
                for s in range(10):
                    bm.validate_plan(bm.plan_step(I, J, s), I, J)

    @pytest.mark.parametrize("gi,gj", [(0, 1), (1, 0)])
    def test_rejects_degenerate(self, gi, gj):
        with pytest.raises(ValueError):
            bm.plan_step(gi, gj, 0)

    def test_rejects_negative_step(self):
        with pytest.raises(ValueError):
            bm.plan_step(2, 2, -1)

    def test_validator_messages(self):
        with pytest.raises(ValueError, match=r"never schedules block \(0, 1\)"):
            bm.validate_plan(bm.StepPlan(2, 2, (bm.Batch(((0, 0), (1, 1))),)), 2, 2)
        with pytest.raises(ValueError, match="scheduled twice"):
            bm.validate_plan(bm.StepPlan(1, 2, (bm.Batch(((0, 0),)), bm.Batch(((0, 0),)),
                                               bm.Batch(((0, 1),)))), 1, 2)
        with pytest.raises(ValueError, match="block-row 0 appears twice"):
            bm.validate_plan(bm.StepPlan(2, 2, (bm.Batch(((0, 0), (0, 1))),
                                               bm.Batch(((1, 0), (1, 1))))), 2, 2)
        with pytest.raises(ValueError, match="block-col 0 appears twice"):
            bm.validate_plan(bm.StepPlan(2, 2, (bm.Batch(((0, 0), (1, 0))),
                                               bm.Batch(((0, 1), (1, 1))))), 2, 2)
        with pytest.raises(ValueError, match=r"\(1, 5\) outside"):
            bm.validate_plan(bm.StepPlan(2, 2, (bm.Batch(((0, 0), (1, 5))),)), 2, 2)


class TestGrid:
    def test_split_bounds(self, golden):
        assert bm.split_bounds(10, 3).tolist() == golden["hand"]["split_bounds_10_3"]
        assert bm.split_bounds(8, 4).tolist() == [0, 2, 4, 6, 8]
        assert bm.split_bounds(5, 1).tolist() == [0, 5]
        with pytest.raises(ValueError, match="non-empty"):
            bm.split_bounds(3, 4)

    @given(st.integers(1, 500), st.integers(1, 32))
    def test_balanced_cover(self, n, parts):
        if parts > n:
            return
        b = bm.split_bounds(n, parts)
        sizes = np.diff(b)
        assert b[0] == 0 and b[-1] == n and sizes.min() >= 1
        assert sizes.max() - sizes.min() <= 1
        assert all(sizes[i] >= sizes[i + 1] for i in range(len(sizes) - 1))

    def test_locate(self, golden):
        assert list(bm.locate(bm.make_grid(1024, 1024, 32, 32), 100, 200)) == golden["hand"]["locate"]
        g = bm.make_grid(10, 7, 3, 2)
        for r in range(10):
            for c in range(7):
                bi, bj, lr, lc = bm.locate(g, r, c)
                assert g.row_bounds[bi] + lr == r and g.col_bounds[bj] + lc == c
        with pytest.raises(IndexError):
            bm.locate(bm.make_grid(4, 4, 2, 2), 4, 0)

    def test_make_grid_validation(self):
        with pytest.raises(ValueError):
            bm.make_grid(4, 4, 5, 1)
        with pytest.raises(ValueError):
            bm.make_grid(4, 4, 1, 0)


class TestCoreTypes:
    def test_schedules_roundtrip(self):
        for text in ("const:3", "inc:2,5", "dec:8", "adaptive:4", "converge:0.001"):
            assert bm.format_schedule(bm.parse_schedule(text)) == text
        for bad in ("const", "const:x", "inc:3", "nope:1", "const:0", "converge:0"):
            with pytest.raises(ValueError):
                bm.parse_schedule(bad)

    def test_resolve_inner_iters(self):
        r = bm.resolve_inner_iters
        assert [r(bm.IncreasingEvery(2, 3), s) for s in range(1, 9)] == [1, 1, 2, 2, 3, 3, 3, 3]
        assert [r(bm.Decreasing(4), s) for s in range(1, 7)] == [4, 3, 2, 1, 1, 1]
        assert r(bm.AdaptiveDecreasing(8), 2, 0.5) == 4
        assert r(bm.AdaptiveDecreasing(8), 2, 0.0) == 1
        assert r(bm.ConvergeEachBlock(0.1), 1) is None
        with pytest.raises(ValueError):
            r(bm.Constant(1), 0)

    def test_config_validation(self):
        bm.TrainConfig()
        for kw in (dict(k=0), dict(alpha=0), dict(beta=-1), dict(delta=-1), dict(outer_steps=0),
                   dict(grid_i=0), dict(workers=0)):
            with pytest.raises(ValueError):
                bm.TrainConfig(**kw)

    def test_dataset_validation(self):
        with pytest.raises(ValueError):
            bm.RatingsDataset(-1, 2, [], [], [])
        with pytest.raises(ValueError):
            bm.RatingsDataset(2, 2, [0], [0, 1], [1.0])
        d = bm.RatingsDataset.from_triples(2, 2, [(0, 0, 3.0)])
        bm.validate_dataset(d)
        with pytest.raises(bm.DataError, match="outside"):
            bm.validate_dataset(bm.RatingsDataset.from_triples(2, 2, [(2, 0, 3.0)]))
        with pytest.raises(bm.DataError, match="duplicate"):
            bm.validate_dataset(bm.RatingsDataset.from_triples(2, 2, [(0, 0, 1.0), (0, 0, 2.0)]))
        with pytest.raises(bm.DataError, match="non-finite"):
            bm.validate_dataset(bm.RatingsDataset.from_triples(2, 2, [(0, 0, np.inf)]))
        with pytest.raises(ValueError):
            d.values[0] = 1.0

    def test_trace_monotone(self):
        t = bm.ConvergenceTrace()
        t.append(bm.TraceStep(1, 1.0, None, 0.0, 1))
        with pytest.raises(ValueError):
            t.append(bm.TraceStep(1, 1.0, None, 0.0, 1))
        with pytest.raises(ValueError):
            t.append(bm.TraceStep(2, -1.0, None, 0.0, 1))

    def test_init_factors(self, golden):
        m = bm.init_factors(943, 1682, 30, 0)
        assert sha(m.u) == golden["partition"]["init_943_1682_30_0"]["u"]
        assert sha(m.v) == golden["partition"]["init_943_1682_30_0"]["v"]
        assert bm.init_factors(100, 100, 25, 1).u.max() < 0.2
        with pytest.raises(ValueError):
            bm.init_factors(0, 1, 1, 0)

    def test_accumulators(self):
        a, b = bm.RmseAccumulator(9.0, 1), bm.RmseAccumulator(16.0, 1)
        assert bm.merge(a, b) == bm.RmseAccumulator(25.0, 2)
        assert bm.finalize(bm.RmseAccumulator()) == 0.0
        with pytest.raises(ValueError):
            bm.RmseAccumulator(-1.0, 0)

    def test_block_task_validation(self):
        with pytest.raises(ValueError, match="converge_tol"):
            bm.BlockTask(0, 0, np.array([0]), np.array([0]), np.array([1.0]), np.ones((1, 1)),
                         np.ones((1, 1)), 0.1, 0.0, inner_iters=None, converge_tol=0.0)
        with pytest.raises(ValueError, match="inner_iters"):
            bm.BlockTask(0, 0, np.array([0]), np.array([0]), np.array([1.0]), np.ones((1, 1)),
                         np.ones((1, 1)), 0.1, 0.0, inner_iters=0)


class TestGenerators:
    def test_dense_and_sparse(self, golden, dense32, dense64, dense256):
        for name, d in (("dense32", dense32), ("dense64", dense64), ("dense256", dense256)):
            g = golden["partition"][name]
            assert (sha(d.rows), sha(d.cols), sha(d.values)) == (g["rows"], g["cols"], g["vals"])
        sp = bm.gen_synthetic(bm.SyntheticSpec(40, 30, 1, 5, seed=3, density=0.3))
        g = golden["partition"]["sparse_gen"]
        assert len(sp) == g["n"] and sha(sp.rows) == g["rows"] and sha(sp.values) == g["vals"]

    def test_standin_and_split(self, golden, standin):
        g = golden["partition"]["standin"]
        assert sha(standin.rows) == g["in_rows"] and sha(standin.values) == g["in_vals"]
        tr, te = bm.split(standin, 0.2, seed=0)
        s = golden["partition"]["standin_split"]
        assert sha(tr.rows) == s["train_rows"] and sha(te.cols) == s["test_cols"]
        assert sha(te.values) == s["test_vals"]

    def test_feistel_is_a_sampling_without_replacement(self):
        for total, count in ((97, 97), (1000, 640), (12345, 100), (2**20 + 3, 5000)):
            cells = workloads.feistel_cells(total, count, seed=5)
            assert cells.min() >= 0 and cells.max() < total
            assert len(np.unique(cells)) == count
        a = workloads.feistel_cells(10**6, 1000, seed=1)
        b = np.concatenate([workloads.feistel_cells(10**6, 500, seed=1),
                            workloads.feistel_cells(10**6, 500, seed=1, start=500)])
        assert np.array_equal(a, b)

    def test_lowrank_shape(self):
        r, c, v = workloads.lowrank(600, 370, 10_000, seed=0)
        assert len(np.unique(r * 370 + c)) == 10_000
        assert v.min() >= 1 and v.max() <= 5 and np.all(v == np.rint(v))
        assert not np.all(np.diff(r * 370 + c) > 0)  # not row-major
