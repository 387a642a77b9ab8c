"""Out-of-core mode: ratings in pinned host memory, streamed
through a ring of device slots each step.  Same algorithm as the in-core
path -- checked against the oracle per epoch (1e-3 absolute) with budgets
that force many pieces per stratum, plus streamed-byte accounting."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from oracle import oracle as O
from paper_2304_13724_b200 import workloads

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _c2_like(nnz=400_000):
    r, c, v = workloads.lowrank(6040, 3706, nnz, seed=3)
    return bm.RatingsDataset(6040, 3706, r, c, v)


@pytest.mark.parametrize("budget_frac,slots,half", [(0.05, 2, False), (0.2, 3, False),
                                                    (0.5, 4, False), (0.2, 3, True)])
def test_stream_matches_oracle(budget_frac, slots, half):
    d = _c2_like()
    if half:  # half-star ratings: not 1-byte integers, fp32 values in the records
        d = bm.RatingsDataset(d.n, d.m, d.rows, d.cols, d.values - 0.5)
    tr, te = bm.split(d, 0.2, seed=0)
    cfg = bm.TrainConfig(k=32, outer_steps=5, grid_i=8, grid_j=8)
    opts = bm.EngineOptions(device_rating_budget=int(12 * len(tr) * budget_frac),
                            stream_slots=slots)
    blocked = bm.partition(tr, 8, 8, options=opts)
    assert blocked.engine.streaming
    res = bm.train_blocked(tr, cfg, te, early_stop=False, timing=False, blocked=blocked)
    _, _, otr, _ = O.train_blocked(tr.n, tr.m, tr.rows, tr.cols, tr.values, k=32, outer_steps=5,
                                   grid_i=8, grid_j=8, test=(te.rows, te.cols, te.values),
                                   early_stop=False, nthreads=8)
    dtr = np.abs(np.array([s.train_rmse for s in res.trace]) - [s["train_rmse"] for s in otr])
    dte = np.abs(np.array([s.test_rmse for s in res.trace]) - [s["test_rmse"] for s in otr])
    assert dtr.max() <= TOL and dte.max() <= TOL
    # every epoch streams every rating once, as packed records: block-local
    # row << cbits | col (4 B) and the value -- a 1-byte code for integer
    # ratings 0..255, else fp32
    per = 8.0 if half else 5.0
    assert blocked.engine.streamed_bytes() == pytest.approx(per * len(tr) * 5)


def test_stream_partition_export_and_sse_only_pass():
    d = _c2_like(100_000)
    ref = O.partition(d.rows, d.cols, d.values, d.n, d.m, 4, 4)
    b = bm.partition(d, 4, 4, options=bm.EngineOptions(device_rating_budget=12 * 40_000))
    assert b.engine.streaming
    assert np.array_equal(b._rows, ref["rows"]) and np.array_equal(b._values, ref["values"])
    # adaptive schedule needs RMSE_0: the zero-sweep streamed SSE pass
    cfg = bm.TrainConfig(k=16, outer_steps=3, grid_i=4, grid_j=4, alpha=1e-3,
                         inner_schedule=bm.AdaptiveDecreasing(4))
    res = bm.train_blocked(d, cfg, early_stop=False, blocked=b)
    u, v, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=16, outer_steps=3,
                                   alpha=1e-3, grid_i=4, grid_j=4, schedule="adaptive:4",
                                   early_stop=False, nthreads=8)
    assert [s.inner_iters for s in res.trace] == [s["inner_iters"] for s in otr]
    got = np.array([s.train_rmse for s in res.trace])
    assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= TOL


def test_stream_rejects_slot_smaller_than_a_block():
    d = _c2_like(50_000)
    with pytest.raises(ValueError, match="largest block"):
        bm.partition(d, 2, 2, options=bm.EngineOptions(device_rating_budget=12 * 3000))


@pytest.mark.parametrize("streamed", [False, True])
def test_l2_waves_match_oracle(streamed):
    """l2_wave_bytes small enough that every stratum runs as one wave per
    block (in core) / one piece per block (streamed): still the reference
    algorithm, per-epoch RMSE within 1e-3 of the oracle."""
    d = _c2_like()
    cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8)
    opts = bm.EngineOptions(l2_wave_bytes=1,
                            device_rating_budget=(12 * len(d) // 2) if streamed else None)
    blocked = bm.partition(d, 8, 8, options=opts)
    assert blocked.engine.streaming == streamed
    res = bm.train_blocked(d, cfg, early_stop=False, timing=False, blocked=blocked)
    _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=4,
                                   grid_i=8, grid_j=8, early_stop=False, nthreads=8)
    got = np.array([s.train_rmse for s in res.trace])
    assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= TOL


@pytest.mark.parametrize("tol", [0.05, 0.005])
def test_stream_converge_schedule_matches_oracle(tol):
    """ConvergeEachBlock out of core: each piece is copied into a slot once and
    its blocks sweep until their RMSE improves by less than tol (cap 100);
    trace within 1e-3 of the oracle, the same per-step sweep counts within one
    (a block's improvement can sit at the tolerance), capped blocks counted."""
    d = _c2_like(200_000)
    cfg = bm.TrainConfig(k=32, outer_steps=3, grid_i=8, grid_j=8,
                         inner_schedule=bm.ConvergeEachBlock(tol))
    opts = bm.EngineOptions(device_rating_budget=int(12 * len(d) * 0.1), stream_slots=3)
    blocked = bm.partition(d, 8, 8, options=opts)
    assert blocked.engine.streaming
    res = bm.train_blocked(d, cfg, early_stop=False, timing=False, blocked=blocked)
    _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=3,
                                   grid_i=8, grid_j=8, schedule=f"converge:{tol}",
                                   early_stop=False, nthreads=8)
    dtr = np.abs(np.array([s.train_rmse for s in res.trace]) - [s["train_rmse"] for s in otr])
    assert dtr.max() <= TOL
    assert all(abs(a.inner_iters - b["inner_iters"]) <= 1 for a, b in zip(res.trace, otr))
    assert all(s.inner_iters >= 1 for s in res.trace)


@pytest.mark.parametrize("budget_ratings", [3_000, 9_000, 19_000])
def test_out_of_core_partition_bit_identical(budget_ratings):
    """bgmf_partition_ooc (row blocks in chunks under the device budget,
    straight into the pinned streaming layout) yields exactly the in-core
    partition: offsets, order, local rows and cols -- the reference's lexsort
    order, reference partition.py:112-136."""
    n, m, nnz, P = 3000, 2000, 60_000, 6
    g = np.random.default_rng(budget_ratings)
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    r[::97] = r[::89][: len(r[::97])]  # some duplicates
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    ref = bm.Engine()
    ref.partition(r, c, v, n, m, P, P)
    want = ref.export_partition()
    ref.close()
    eng = bm.Engine(bm.EngineOptions(device_rating_budget=12 * budget_ratings * 3, stream_slots=3))
    eng.partition(r, c, v, n, m, P, P)
    assert eng.streaming
    got = eng.export_partition()
    eng.close()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_out_of_core_partition_peak_memory():
    """The device pool's high-water mark of an out-of-core partition stays
    within the budget (plus the slot ring and a few MB of fixed scratch),
    ~an order of magnitude under the in-core partition of the same data."""
    n, m, nnz, P = 200_000, 50_000, 4_000_000, 16
    g = np.random.default_rng(7)
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    inc = bm.Engine()
    inc.mem_stats(reset=True)
    base, _ = inc.mem_stats()
    inc.partition(r, c, v, n, m, P, P)
    _, high_in = inc.mem_stats()
    inc.close()
    budget = 16 << 20  # 16 MB: ~250k ratings of chunk temporaries, 1/16 of the data
    eng = bm.Engine(bm.EngineOptions(device_rating_budget=budget, stream_slots=3))
    eng.mem_stats(reset=True)
    base2, _ = eng.mem_stats()
    eng.partition(r, c, v, n, m, P, P)
    _, high = eng.mem_stats()
    eng.close()
    slots = 3 * (budget // 36) * 8
    print(f"in-core partition peak {(high_in - base) / 2**20:.1f} MB, out-of-core "
          f"{(high - base2) / 2**20:.1f} MB (budget {budget / 2**20:.0f} MB + slots "
          f"{slots / 2**20:.1f} MB)")
    assert high - base2 <= budget + slots + (4 << 20)
    assert high - base2 < (high_in - base) / 4


def test_out_of_core_pinned_cache_reuse():
    """A closed out-of-core context leaves its pinned layout in the process
    cache; the next partition of the same size reuses it (no re-pinning) and
    is still bit-identical; bgmf_release_host_cache empties the cache."""
    from paper_2304_13724_b200.device import release_host_cache
    n, m, nnz, P = 3000, 2000, 80_000, 5
    g = np.random.default_rng(9)
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    outs = []
    for _ in range(3):
        eng = bm.Engine(bm.EngineOptions(device_rating_budget=12 * 6000 * 3, stream_slots=3))
        eng.partition(r, c, v, n, m, P, P)
        assert eng.streaming
        outs.append(eng.export_partition())
        eng.close()
    for got in outs[1:]:
        for a, b in zip(got, outs[0]):
            assert np.array_equal(a, b)
    release_host_cache()
    release_host_cache()  # idempotent
