"""GPU partitioner: bit-exact with the reference BlockedDataset
(partition.py:112-136) -- golden arrays, standin hashes, oracle at C2/C3
sizes, and full-size (C4) properties."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from helpers import sha
from oracle import oracle as O
from paper_2304_13724_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["d32_3x5", "d32_4x4", "sparse_6x5", "sparse_1x1", "dup_2x2",
                                  "six_3x3"])
def test_golden_arrays(golden, partition_cases, name):
    meta, P = golden["partition"][name], partition_cases
    d = bm.RatingsDataset(meta["n"], meta["m"], P[name + "_in_rows"], P[name + "_in_cols"],
                          P[name + "_in_vals"])
    b = bm.partition(d, meta["I"], meta["J"])
    assert np.array_equal(b._offsets, P[name + "_offsets"])
    assert np.array_equal(b._rows, P[name + "_rows"])
    assert np.array_equal(b._cols, P[name + "_cols"])
    assert np.array_equal(b._values, P[name + "_vals"])


@pytest.mark.parametrize("grid", ["4x4", "8x8", "3x7"])
def test_standin_hashes(golden, standin, grid):
    h = golden["partition"]["standin"]["partitions"][grid]
    I, J = map(int, grid.split("x"))
    b = bm.partition(standin, I, J)
    assert sha(b._offsets) == h["offsets"]
    assert sha(b._rows) == h["rows"]
    assert sha(b._cols) == h["cols"]
    assert sha(b._values) == h["values"]
    assert b.counts.tolist() == h["counts"]


def test_reference_partition_behaviour(dense32):
    b = bm.partition(dense32, 4, 4)
    assert b.counts.sum() == len(dense32)
    blk = b.block(2, 1)
    keys = list(zip(blk.rows, blk.cols))
    assert keys == sorted(keys)
    with pytest.raises(ValueError):
        b.block(0, 0).values[0] = 0.0
    with pytest.raises(IndexError):
        b.block(4, 0)
    with pytest.raises(ValueError, match="grid is"):
        bm.block_dataset(dense32, bm.make_grid(33, 32, 2, 2))
    seen = set()
    for blk in bm.partition(dense32, 3, 5):
        for lr, lc, v in zip(blk.rows, blk.cols, blk.values):
            seen.add((blk.row_start + lr, blk.col_start + lc, v))
    assert seen == set(zip(dense32.rows, dense32.cols, dense32.values))


def test_empty_and_degenerate():
    d = bm.RatingsDataset.from_triples(6, 6, [(0, 0, 1.0), (5, 5, 2.0)])
    assert bm.partition(d, 3, 3).counts.tolist() == [[1, 0, 0], [0, 0, 0], [0, 0, 1]]
    e = bm.RatingsDataset.from_triples(4, 4, [])
    b = bm.partition(e, 2, 2)
    assert b.counts.sum() == 0 and len(b.block(1, 1)) == 0
    one = bm.RatingsDataset.from_triples(1, 1, [(0, 0, 3.0)])
    assert bm.partition(one, 1, 1).block(0, 0).values.tolist() == [3.0]
    # grid as fine as the matrix: every slab one index wide
    d = bm.gen_synthetic(bm.SyntheticSpec(7, 5, 1, 5, seed=2, density=0.6))
    ref = O.partition(d.rows, d.cols, d.values, 7, 5, 7, 5)
    b = bm.partition(d, 7, 5)
    assert np.array_equal(b._offsets, ref["offsets"]) and np.array_equal(b._rows, ref["rows"])


def test_out_of_range_index_is_a_data_error():
    d = bm.RatingsDataset(4, 4, [0, 4], [0, 1], [1.0, 2.0])
    with pytest.raises(bm.DataError, match="outside"):
        bm.partition(d, 2, 2)


def test_duplicates_keep_input_order():
    rows = np.array([3, 1, 3, 3, 0, 1, 3, 3])
    cols = np.array([2, 0, 2, 1, 4, 0, 2, 2])
    d = bm.RatingsDataset(5, 5, rows, cols, np.arange(8.0))
    ref = O.partition(d.rows, d.cols, d.values, 5, 5, 2, 2)
    b = bm.partition(d, 2, 2)
    assert np.array_equal(b._values, ref["values"])


@pytest.mark.parametrize("grid", [(8, 8), (5, 11), (1, 1), (16, 3)])
def test_matches_oracle_c2(grid):
    r, c, v = workloads.lowrank(6040, 3706, 1_000_000, seed=1)
    d = bm.RatingsDataset(6040, 3706, r, c, v)
    ref = O.partition(r, c, v, 6040, 3706, *grid)
    b = bm.partition(d, *grid)
    for mine, theirs in (("_offsets", "offsets"), ("_rows", "rows"), ("_cols", "cols"),
                         ("_values", "values")):
        assert np.array_equal(getattr(b, mine), ref[theirs]), mine


@pytest.mark.slow
def test_matches_oracle_c3():
    w = workloads.CONFIGS["C3"]
    r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=0)
    ref = O.partition(r, c, v, w.n, w.m, 8, 8)
    b = bm.partition(bm.RatingsDataset(w.n, w.m, r, c, v), 8, 8)
    assert np.array_equal(b._offsets, ref["offsets"])
    assert np.array_equal(b._rows, ref["rows"])
    assert np.array_equal(b._cols, ref["cols"])
    assert np.array_equal(b._values, ref["values"])
    assert np.array_equal(b.order, np.lexsort((c, r, _block_ids(r, c, w.n, w.m, 8, 8))))


def _block_ids(r, c, n, m, I, J):
    rb, cb = bm.split_bounds(n, I), bm.split_bounds(m, J)
    return (np.searchsorted(rb, r, side="right") - 1) * J + np.searchsorted(cb, c, side="right") - 1


@pytest.mark.slow
def test_c4_full_size_properties():
    """C4 (100M ratings, 16x16): size-independent invariants of the partition."""
    w = workloads.CONFIGS["C4"]
    r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=0)
    b = bm.partition(bm.RatingsDataset(w.n, w.m, r, c, v), 16, 16)
    off, order, lr, lc = b.engine.export_partition()
    assert off[0] == 0 and off[-1] == w.nnz and np.all(np.diff(off) >= 0)
    # order is a permutation and maps back to the source cells
    assert np.array_equal(np.bincount(order, minlength=w.nnz), np.ones(w.nnz, np.int64))
    bid = np.repeat(np.arange(256), np.diff(off))
    rb, cb = bm.split_bounds(w.n, 16), bm.split_bounds(w.m, 16)
    assert np.array_equal(rb[bid // 16] + lr, r[order])
    assert np.array_equal(cb[bid % 16] + lc, c[order])
    # row-major within every block
    key = (bid.astype(np.int64) << 40) | (lr << 20) | lc
    assert np.all(np.diff(key) > 0)
    counts = np.bincount(_block_ids(r, c, w.n, w.m, 16, 16), minlength=256)
    assert np.array_equal(np.diff(off), counts)


def test_partition_rows_keeps_only_the_row_range():
    """bgmf_partition_rows == bgmf_partition of the pre-filtered entries
    (offsets, local coordinates, values), and still range-checks every entry."""
    g = np.random.default_rng(3)
    n, m, nnz = 1000, 700, 50_000
    cells = g.choice(n * m, nnz, replace=False)
    r, c = cells // m, cells % m
    v = g.integers(1, 6, nnz).astype(np.float64)
    for lo, hi in ((0, 1000), (250, 500), (0, 1), (999, 1000), (400, 400)):
        a, b = bm.Engine(), bm.Engine()
        a.partition(r, c, v, n, m, 4, 3, row_range=(lo, hi))
        keep = (r >= lo) & (r < hi)
        b.partition(r[keep], c[keep], v[keep], n, m, 4, 3)
        oa, _, ra, ca = a.export_partition()
        ob, _, rb_, cb = b.export_partition()
        assert np.array_equal(oa, ob) and a.nnz == int(keep.sum())
        assert np.array_equal(ra, rb_) and np.array_equal(ca, cb)
    bad = r.copy()
    bad[123] = n + 5
    with pytest.raises(bm.DataError, match="entry 123"):
        bm.Engine().partition(bad, c, v, n, m, 4, 3, row_range=(0, 10))


@pytest.mark.parametrize("options", [None, bm.EngineOptions(exact=True)], ids=["fast", "exact"])
@pytest.mark.parametrize("shape", [(6040, 3706, 8, 8), (6040, 3706, 2, 3),
                                   (2**31 - 1, 2**30, 1, 1), (2**31 - 1, 2**31 - 1, 3, 2)],
                         ids=["c2-embedded", "c2-8bit", "wide-1x1", "wide-3x2"])
def test_key_layouts_match_oracle(shape, options):
    """Both sort layouts: the source index in the key's spare low bits with
    the fp32 value as payload (fast mode, key + index <= 64 bits) and the
    index as payload with a gather (exact mode, or keys too wide: 2^31-row
    matrices), with duplicate cells, against the oracle's lexsort order."""
    n, m, I, J = shape
    g = np.random.default_rng(n % 1000 + I)
    nnz = 60_000
    r = g.integers(0, n, nnz)
    c = g.integers(0, m, nnz)
    dup, at = g.integers(0, nnz, 5_000), g.integers(0, nnz, 5_000)
    r[at], c[at] = r[dup], c[dup]  # repeated cells keep input order
    v = g.integers(1, 6, nnz).astype(np.float64) + g.random(nnz)
    ref = O.partition(r, c, v, n, m, I, J)
    b = bm.partition(bm.RatingsDataset(n, m, r, c, v), I, J, options)
    assert np.array_equal(b._offsets, ref["offsets"])
    assert np.array_equal(b._rows, ref["rows"])
    assert np.array_equal(b._cols, ref["cols"])
    assert np.array_equal(b._values, ref["values"])
    assert np.array_equal(b.order, np.lexsort((c, r, _block_ids(r, c, n, m, I, J))))



@pytest.mark.parametrize("kind", ["ints", "floats"])
def test_device_values_are_the_narrowed_inputs(kind):
    """bgmf_partition_values: the fp32 values the kernels read, in partition
    order, are the fp64 inputs narrowed (bit-exact, -0.0 kept); indices
    bit-equal to the oracle.  4 M entries = several staging chunks."""
    from paper_2304_13724_b200.device import Engine, EngineOptions
    g = np.random.default_rng(5)
    n, m, nnz = 480_000, 17_800, 4_000_000
    r = g.integers(0, n, nnz)
    c = g.integers(0, m, nnz)
    v = np.rint(g.uniform(0, 255, nnz)) if kind == "ints" else g.normal(3.0, 2.0, nnz)
    v[:4] = [-0.0, 0.5, 1e9, 256.0]
    eng = Engine(EngineOptions())
    eng.partition(r, c, v, n, m, 8, 8)
    off, order, lr, lc = eng.export_partition()
    vals = eng.partition_values()
    eng.close()
    assert np.array_equal(vals.view(np.int64),
                          v[order].astype(np.float32).astype(np.float64).view(np.int64))
    P = O.partition(r, c, v, n, m, 8, 8)
    assert np.array_equal(off, P["offsets"])
    assert np.array_equal(lr, P["rows"]) and np.array_equal(lc, P["cols"])
