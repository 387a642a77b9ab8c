"""init_factors on the device: numpy's PCG64 stream reproduced bit-for-bit
(reference core.py:179-193) -- fp64 in exact mode, its fp32 rounding in fast
mode."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,k,seed", [(1, 1, 1, 0), (943, 1682, 30, 0), (64, 64, 10, 7),
                                        (1000, 37, 128, 123456789), (5, 3, 513, 2)])
def test_device_init_bit_identical(n, m, k, seed):
    d = bm.RatingsDataset(n, m, [0], [0], [1.0])
    ref = bm.init_factors(n, m, k, seed)
    ex = bm.Engine(bm.EngineOptions(exact=True))
    ex.partition(d.rows, d.cols, d.values, n, m, 1, 1)
    ex.init_factors(n, m, k, seed)
    u, v = ex.get_factors()
    assert np.array_equal(u, ref.u) and np.array_equal(v, ref.v)
    if k <= 512:
        fa = bm.Engine()
        fa.partition(d.rows, d.cols, d.values, n, m, 1, 1)
        fa.init_factors(n, m, k, seed)
        u, v = fa.get_factors()
        assert np.array_equal(u, ref.u.astype(np.float32).astype(np.float64))
        assert np.array_equal(v, ref.v.astype(np.float32).astype(np.float64))


def test_device_synth_cells_match_numpy_feistel():
    """bgmf_synth samples the same cells as workloads.feistel_cells (integer
    math), values on the 1..5 scale; bgmf_synth_partition partitions them."""
    from paper_2304_13724_b200 import _native as N
    from paper_2304_13724_b200 import workloads

    L = N.load()
    n, m, nnz, seed = 6040, 3706, 200_000, 11
    rows = np.empty(nnz, np.int64)
    cols = np.empty(nnz, np.int64)
    vals = np.empty(nnz, np.float64)
    N.check(L.bgmf_synth(n, m, nnz, 0, seed, N.ptr(rows, N._i64p), N.ptr(cols, N._i64p),
                         N.ptr(vals, N._f64p)))
    cells = workloads.feistel_cells(n * m, nnz, seed)
    assert np.array_equal(rows * m + cols, cells)
    assert vals.min() >= 1 and vals.max() <= 5 and np.all(vals == np.rint(vals))
    assert 2.5 < vals.mean() < 4.5
    eng = bm.Engine()
    N.check(L.bgmf_synth_partition(eng._h, n, m, nnz, seed, 8, 8), eng._h)
    eng.n, eng.m, eng.nnz, eng.I, eng.J = n, m, nnz, 8, 8
    off, order, lr, lc = eng.export_partition()
    from oracle import oracle as O
    ref = O.partition(rows, cols, vals, n, m, 8, 8)
    assert np.array_equal(off, ref["offsets"]) and np.array_equal(lr, ref["rows"])
    assert np.array_equal(lc, ref["cols"]) and np.array_equal(vals[order], ref["values"])
