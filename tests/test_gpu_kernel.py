"""Single-block kernel boundary (_kernels.sgd_sweeps / sgd_converge /
block_sse replacements): the stateless C-ABI drop-ins run on the GPU in fp64
and must be bit-identical with the reference, including the reference's own
hand-computed unit tests (test_kernel.py)."""

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from paper_2304_13724_b200.kernel import CONVERGE_CAP

pytestmark = pytest.mark.gpu


def one_entry_task(alpha=0.1, beta=0.5, inner_iters=1, converge_tol=0.0):
    return bm.BlockTask(bi=0, bj=0, rows=np.array([0]), cols=np.array([0]),
                        values=np.array([2.0]), u_slice=np.array([[1.0]]),
                        v_slice=np.array([[1.0]]), alpha=alpha, beta=beta,
                        inner_iters=inner_iters, converge_tol=converge_tol)


def test_single_entry_hand_computed():
    task = one_entry_task()
    stats = bm.sgd_block(task)
    expected = 1.0 + 0.1 * (2.0 * 1.0 * 1.0 - 0.5 * 1.0)
    assert task.u_slice[0, 0] == expected and task.v_slice[0, 0] == expected
    assert stats.sse_before == 1.0
    assert stats.sse_after == pytest.approx((2.0 - expected * expected) ** 2, rel=1e-15)
    assert stats.entries == 1 and stats.iters_used == 1


def test_pre_update_vectors():
    task = bm.BlockTask(bi=0, bj=0, rows=np.array([0]), cols=np.array([0]),
                        values=np.array([3.0]), u_slice=np.array([[2.0]]),
                        v_slice=np.array([[0.5]]), alpha=0.1, beta=0.0, inner_iters=1)
    bm.sgd_block(task)
    e = 3.0 - 2.0 * 0.5
    assert task.u_slice[0, 0] == 2.0 + 0.1 * 2.0 * e * 0.5
    assert task.v_slice[0, 0] == 0.5 + 0.1 * 2.0 * e * 2.0


def test_spec_examples():
    # x=4 -> 1.6; beta=.5 -> 1.55
    for beta, want in ((0.0, 1.6), (0.5, 1.55)):
        t = bm.BlockTask(0, 0, np.array([0]), np.array([0]), np.array([4.0]),
                         np.array([[1.0]]), np.array([[1.0]]), 0.1, beta, 1)
        bm.sgd_block(t)
        assert t.u_slice[0, 0] == pytest.approx(want, rel=1e-15)


def test_row_major_order_observable():
    rows, cols, values = np.array([0, 1]), np.array([0, 0]), np.array([1.0, 2.0])
    u, v = np.array([[0.5], [0.5]]), np.array([[0.5]])
    task = bm.BlockTask(0, 0, rows, cols, values, u, v, 0.1, 0.0, 1)
    bm.sgd_block(task)
    uu, vv = np.array([0.5, 0.5]), 0.5
    for i in range(2):
        e = values[i] - uu[i] * vv
        ui = uu[i] + 0.1 * 2.0 * e * vv
        vv = vv + 0.1 * 2.0 * e * uu[i]
        uu[i] = ui
    assert np.array_equal(task.u_slice[:, 0], uu) and task.v_slice[0, 0] == vv


@pytest.mark.parametrize("t", range(12))
def test_golden_sweeps_and_converge(kernel_cases, t):
    K, p = kernel_cases, f"c{t}_"
    alpha, beta, iters, tol = K[p + "params"]
    u, v = K[p + "u"].copy(), K[p + "v"].copy()
    st = bm.sgd_block(bm.BlockTask(0, 0, K[p + "rows"], K[p + "cols"], K[p + "vals"], u, v,
                                   alpha, beta, int(iters)))
    assert np.array_equal(u, K[p + "u_after"]) and np.array_equal(v, K[p + "v_after"])
    assert (st.sse_before, st.sse_after) == tuple(K[p + "out"][:2])
    u, v = K[p + "u"].copy(), K[p + "v"].copy()
    st = bm.sgd_block(bm.BlockTask(0, 0, K[p + "rows"], K[p + "cols"], K[p + "vals"], u, v,
                                   alpha, beta, None, tol))
    ref = K[p + "out_conv"]
    assert np.array_equal(u, K[p + "u_conv"]) and np.array_equal(v, K[p + "v_conv"])
    assert (st.sse_before, st.sse_after, st.iters_used, int(st.capped)) == \
        (ref[0], ref[1], ref[2], ref[3])


def test_block_sse_pure(kernel_cases):
    K = kernel_cases
    for t in range(12):
        p = f"c{t}_"
        task = bm.BlockTask(0, 0, K[p + "rows"], K[p + "cols"], K[p + "vals"], K[p + "u"].copy(),
                            K[p + "v"].copy(), 0.1, 0.0, 1)
        assert bm.block_sse(task) == K[p + "out"][0]
        assert np.array_equal(task.u_slice, K[p + "u"])


def test_multiple_sweeps_descend(dense32):
    block = bm.partition(dense32, 1, 1).block(0, 0)
    model = bm.init_factors(32, 32, 4, seed=0)
    stats = bm.sgd_block(bm.task_from_block(block, model, 1e-3, 1e-2, 5))
    assert stats.sse_after < stats.sse_before and stats.iters_used == 5


def test_empty_block_no_op():
    task = bm.BlockTask(0, 0, np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0),
                        np.ones((2, 2)), np.ones((2, 2)), 0.1, 0.0, 3)
    stats = bm.sgd_block(task)
    assert stats.sse_before == stats.sse_after == 0.0
    assert np.array_equal(task.u_slice, np.ones((2, 2)))


def test_converge_mode():
    stats = bm.sgd_block(one_entry_task(inner_iters=None, converge_tol=1e-4))
    assert 1 <= stats.iters_used < CONVERGE_CAP and not stats.capped
    assert stats.sse_after < stats.sse_before
    stats = bm.sgd_block(one_entry_task(alpha=1e-13, beta=0.0, inner_iters=None,
                                        converge_tol=1e-300))
    assert stats.capped and stats.iters_used == CONVERGE_CAP


def test_divergence_location(kernel_cases, dense32):
    block = bm.partition(dense32, 2, 2).block(1, 0)
    model = bm.init_factors(32, 32, 4, seed=0)
    with pytest.raises(bm.DivergenceError) as info:
        bm.sgd_block(bm.task_from_block(block, model, 1e6, 0.0, 50))
    err = info.value
    ref = kernel_cases["div_out"]
    assert err.block == (1, 0) and (err.entry, err.iteration) == (int(ref[2]), int(ref[3]))
    assert "reduce alpha" in str(err)


def test_slices_alias_the_model(dense32):
    blocked = bm.partition(dense32, 4, 4)
    model = bm.init_factors(32, 32, 2, seed=0)
    block = blocked.block(2, 3)
    task = bm.task_from_block(block, model, 1e-4, 0.0, 1)
    before = model.u.copy()
    bm.sgd_block(task)
    assert not np.array_equal(model.u, before)
    changed = np.flatnonzero(np.any(model.u != before, axis=1))
    assert changed.min() >= block.row_start and changed.max() < block.row_stop
