"""Pin the CPU oracle (oracle/) against the reference's golden vectors.

The fixtures were produced by the unmodified reference package
(tests/golden/make_golden.py); the oracle must reproduce every one of them
bit-for-bit before it is trusted as the checker of the GPU path.
"""

import numpy as np
import pytest

from helpers import config_of, sha, trace_inputs
from oracle import oracle as O

from paper_2304_13724_b200 import workloads


def test_oracle_builds():
    assert O.build().endswith("liboracle.so")


@pytest.mark.parametrize("t", range(12))
def test_sgd_sweeps_bit_exact(kernel_cases, t):
    K, p = kernel_cases, f"c{t}_"
    alpha, beta, iters, _ = K[p + "params"]
    u, v = K[p + "u"].copy(), K[p + "v"].copy()
    out = O.sgd_sweeps(K[p + "rows"], K[p + "cols"], K[p + "vals"], u, v, alpha, beta, int(iters))
    assert np.array_equal(u, K[p + "u_after"])
    assert np.array_equal(v, K[p + "v_after"])
    assert np.array_equal(np.array(out, float), K[p + "out"])


@pytest.mark.parametrize("t", range(12))
def test_sgd_converge_bit_exact(kernel_cases, t):
    K, p = kernel_cases, f"c{t}_"
    alpha, beta, _, tol = K[p + "params"]
    u, v = K[p + "u"].copy(), K[p + "v"].copy()
    out = O.sgd_converge(K[p + "rows"], K[p + "cols"], K[p + "vals"], u, v, alpha, beta, tol,
                         10_000)
    assert np.array_equal(u, K[p + "u_conv"])
    assert np.array_equal(v, K[p + "v_conv"])
    assert np.array_equal(np.array(out, float), K[p + "out_conv"], equal_nan=True)


def test_block_sse_matches_sweep_before(kernel_cases):
    K = kernel_cases
    for t in range(12):
        p = f"c{t}_"
        s = O.block_sse(K[p + "rows"], K[p + "cols"], K[p + "vals"], K[p + "u"], K[p + "v"])
        assert s == K[p + "out"][0]


def test_divergence_location(kernel_cases, dense32):
    P = O.partition(dense32.rows, dense32.cols, dense32.values, 32, 32, 2, 2)
    b = 1 * 2 + 0
    lo, hi = P["offsets"][b], P["offsets"][b + 1]
    u, v = O.init_factors(32, 32, 4, 0)
    us, vs = u[16:32].copy(), v[0:16].copy()
    out = O.sgd_sweeps(P["rows"][lo:hi], P["cols"][lo:hi], P["values"][lo:hi], us, vs, 1e6, 0.0, 50)
    ref = kernel_cases["div_out"]
    assert out[0] == ref[0] and np.isnan(out[1]) and np.isnan(ref[1])
    assert (out[2], out[3]) == (ref[2], ref[3])


@pytest.mark.parametrize("name", ["d32_3x5", "d32_4x4", "sparse_6x5", "sparse_1x1", "dup_2x2",
                                  "six_3x3"])
def test_partition_bit_exact(golden, partition_cases, name):
    meta, P = golden["partition"][name], partition_cases
    R = O.partition(P[name + "_in_rows"], P[name + "_in_cols"], P[name + "_in_vals"], meta["n"],
                    meta["m"], meta["I"], meta["J"])
    for mine, ref in (("offsets", "offsets"), ("rows", "rows"), ("cols", "cols"),
                      ("values", "vals")):
        assert np.array_equal(R[mine], P[name + "_" + ref]), mine


@pytest.mark.parametrize("grid", ["4x4", "8x8", "3x7"])
def test_partition_standin_hashes(golden, standin, grid):
    h = golden["partition"]["standin"]["partitions"][grid]
    I, J = map(int, grid.split("x"))
    R = O.partition(standin.rows, standin.cols, standin.values, 943, 1682, I, J)
    assert sha(R["offsets"]) == h["offsets"]
    assert sha(R["rows"]) == h["rows"]
    assert sha(R["cols"]) == h["cols"]
    assert sha(R["values"]) == h["values"]
    assert np.diff(R["offsets"]).reshape(I, J).tolist() == h["counts"]


def test_plans_match_reference(golden):
    for key, text in golden["plans"].items():
        I, J, s = map(int, key.split(","))
        got = "\n".join(" ".join(f"({a},{b})" for a, b in batch) for batch in O.plan_step(I, J, s))
        assert got == text, key


TRACES = ["dense64_const1", "dense64_const3", "dense64_dec4", "dense64_inc", "dense64_adaptive",
          "dense64_converge", "dense64_early", "dense64_wide_2x5", "dense64_tall_5x2",
          "dense64_holdout", "c1_k30", "c1_k10", "c1_split"]


@pytest.mark.parametrize("name", TRACES)
def test_train_trace_bit_exact(golden, name):
    meta = golden["traces"][name]
    d, te = trace_inputs(name)
    cfg = config_of(meta)
    test = (te.rows, te.cols, te.values) if te is not None else None
    u, v, trace, stop = O.train_blocked(
        d.n, d.m, d.rows, d.cols, d.values, k=cfg.k, alpha=cfg.alpha, beta=cfg.beta,
        delta=cfg.delta, outer_steps=cfg.outer_steps, schedule=meta["cfg"]["schedule"],
        grid_i=cfg.grid_i, grid_j=cfg.grid_j, seed=cfg.seed, test=test,
        early_stop=meta["early_stop"], nthreads=4)
    assert [s["train_rmse"] for s in trace] == meta["train"]
    assert [s["test_rmse"] for s in trace] == meta["test"]
    assert [s["inner_iters"] for s in trace] == meta["inner"]
    assert [s["capped_blocks"] for s in trace] == meta["capped"]
    assert stop == meta["stop"]
    assert sha(u) == meta["u_sha"] and sha(v) == meta["v_sha"]
    assert O.rmse(u, v, d.rows, d.cols, d.values) == meta["final_rmse"]


def test_threads_do_not_change_results():
    d = workloads.ml100k_dataset()
    outs = []
    for nt in (1, 8):
        u, v, tr, _ = O.train_blocked(943, 1682, d.rows, d.cols, d.values, k=8, outer_steps=3,
                                      grid_i=4, grid_j=4, early_stop=False, nthreads=nt)
        outs.append((sha(u), sha(v), [s["train_rmse"] for s in tr]))
    assert outs[0] == outs[1]


def test_hand_values(golden):
    h = golden["hand"]
    assert O.split_bounds(10, 3).tolist() == h["split_bounds_10_3"]
    u = np.array([[1.0], [2.0]])
    assert O.rmse(u, u, np.array([0, 1]), np.array([0, 1]), np.array([4.0, 8.0])) == h["rmse_hand"]


# ---- verification kernels and baseline trainers ------

@pytest.mark.parametrize("t", range(12))
def test_gradient_steps_bit_exact(baseline_cases, t):
    K, p = baseline_cases, f"g{t}_"
    alpha, beta, iters = K[p + "params"]
    u, v = K[p + "u"].copy(), K[p + "v"].copy()
    out = O.gradient_steps(K[p + "rows"], K[p + "cols"], K[p + "vals"], u, v, alpha, beta,
                           int(iters))
    assert np.array_equal(u, K[p + "u_after"]) and np.array_equal(v, K[p + "v_after"])
    assert np.array_equal(np.array(out, float), K[p + "out"], equal_nan=True)


def test_gradient_steps_divergence(baseline_cases, dense32):
    P = O.partition(dense32.rows, dense32.cols, dense32.values, 32, 32, 1, 1)
    u, v = O.init_factors(32, 32, 4, 0)
    out = O.gradient_steps(P["rows"], P["cols"], P["values"], u, v, 1e6, 0.0, 50)
    ref = baseline_cases["gdiv_out"]
    assert out[0] == ref[0] and np.isnan(out[1]) and (out[2], out[3]) == (ref[2], ref[3])


@pytest.mark.parametrize("t", range(6))
def test_block_gradients_restatement(baseline_cases, t):
    K, p = baseline_cases, f"o{t}_"
    obj, gu, gv = O.block_gradients(K[p + "rows"], K[p + "cols"], K[p + "vals"], K[p + "u"],
                                    K[p + "v"], float(K[p + "beta"][0]))
    assert obj == K[p + "obj"][0]
    assert np.array_equal(gu, K[p + "gu"]) and np.array_equal(gv, K[p + "gv"])


@pytest.mark.parametrize("name", ["cpmf_dense64_w1", "cpmf_dense64_w3", "cpmf_dense64_w4",
                                  "cpmf_dense64_w7", "cpmf_dense64_holdout_w4",
                                  "cpmf_c1_k30_w8"])
def test_sync_parallel_bit_exact(golden, name):
    from helpers import trace_inputs

    meta = golden["baselines"]["traces"][name]
    c = meta["cfg"]
    d, te = trace_inputs(name)
    test = None if te is None else (te.rows, te.cols, te.values)
    u, v, tr, stop = O.train_sync_parallel(d.n, d.m, d.rows, d.cols, d.values, k=c["k"],
                                           alpha=c["alpha"], beta=c["beta"], delta=c["delta"],
                                           outer_steps=c["outer_steps"], seed=c["seed"],
                                           workers=c["workers"], test=test,
                                           early_stop=meta["early_stop"])
    assert [s["train_rmse"] for s in tr] == meta["train"]
    assert stop == meta["stop"]
    assert sha(u) == meta["u_sha"] and sha(v) == meta["v_sha"]
    if te is not None:
        for a, b in zip([s["test_rmse"] for s in tr], meta["test"]):
            assert a == pytest.approx(b, rel=1e-12)


@pytest.mark.parametrize("name", ["cmf_dense64", "cmf_dense64_early", "cmf_c1_k30"])
def test_sequential_is_blocked_1x1(golden, name):
    """baselines.py:62-97: CMF == train_blocked on a 1x1 grid, Constant(1)."""
    from helpers import trace_inputs

    meta = golden["baselines"]["traces"][name]
    c = meta["cfg"]
    d, _ = trace_inputs(name)
    u, v, tr, stop = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=c["k"],
                                     alpha=c["alpha"], beta=c["beta"], delta=c["delta"],
                                     outer_steps=c["outer_steps"], seed=c["seed"],
                                     early_stop=meta["early_stop"])
    assert [s["train_rmse"] for s in tr] == meta["train"]
    assert stop == meta["stop"]
    assert sha(u) == meta["u_sha"] and sha(v) == meta["v_sha"]


@pytest.mark.parametrize("shape", [(2**31 - 1, 2**31 - 1, 3, 2), (2**31 - 1, 2**30, 1, 1),
                                   (100, 70, 3, 4)])
def test_partition_wide_matrices_match_lexsort(shape):
    """The oracle's packed 64-bit key overflows for 2^31-wide matrices; it
    then falls back to a stable comparison sort -- still np.lexsort's order
    (partition.py:124), duplicates in input order."""
    n, m, I, J = shape
    g = np.random.default_rng(3)
    r, c = g.integers(0, n, 20_000), g.integers(0, m, 20_000)
    dup, at = g.integers(0, 20_000, 2_000), g.integers(0, 20_000, 2_000)
    r[at], c[at] = r[dup], c[dup]
    v = g.random(20_000)
    ref = O.partition(r, c, v, n, m, I, J)
    rb, cb = O.split_bounds(n, I), O.split_bounds(m, J)
    bi = np.searchsorted(rb, r, side="right") - 1
    bj = np.searchsorted(cb, c, side="right") - 1
    order = np.lexsort((c, r, bi * J + bj))
    assert np.array_equal(ref["values"], v[order])
    assert np.array_equal(ref["rows"], r[order] - rb[bi[order]])
    assert np.array_equal(ref["cols"], c[order] - cb[bj[order]])
    assert np.array_equal(ref["offsets"], np.concatenate(([0], np.cumsum(
        np.bincount(bi * J + bj, minlength=I * J)))))
