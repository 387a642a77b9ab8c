"""Single-block kernel API (reference ``kernel.py``).

``sgd_block`` is the per-block boundary of the reference (kernel.py:102-139,
which calls numba ``_kernels.sgd_sweeps``/``sgd_converge``).  Here it calls
the stateless C-ABI drop-ins ``bgmf_sgd_sweeps`` / ``bgmf_sgd_converge``,
which run the block on the GPU in fp64 in the reference's exact operation
order, so a single block is bit-identical with the reference.  The
throughput path is not this call but :func:`train_blocked`, which runs whole
strata per launch.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import DivergenceError, FactorModel
from .partition import Block

CONVERGE_CAP = 10_000


@dataclass(frozen=True)
class BlockTask:
    """One kernel invocation (kernel.py:23-54): block-local entries plus
    writable views of the matching U/V slices."""

    bi: int
    bj: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    u_slice: np.ndarray
    v_slice: np.ndarray
    alpha: float
    beta: float
    inner_iters: int | None = 1
    converge_tol: float = 0.0

    def __post_init__(self):
        if self.u_slice.ndim != 2 or self.v_slice.ndim != 2:
            raise ValueError("factor slices must be 2-D")
        if self.u_slice.shape[1] != self.v_slice.shape[1]:
            raise ValueError("factor slices must share latent dimension")
        if self.inner_iters is None:
            if not self.converge_tol > 0:
                raise ValueError("converge mode needs converge_tol > 0")
        elif self.inner_iters < 1:
            raise ValueError("inner_iters must be >= 1")


@dataclass(frozen=True)
class BlockStats:
    sse_before: float
    sse_after: float
    entries: int
    iters_used: int
    capped: bool = False


def task_from_block(block: Block, model: FactorModel, alpha: float, beta: float,
                    inner_iters: int | None, converge_tol: float = 0.0) -> BlockTask:
    return BlockTask(
        bi=block.bi, bj=block.bj, rows=block.rows, cols=block.cols, values=block.values,
        u_slice=model.u[block.row_start:block.row_stop],
        v_slice=model.v[block.col_start:block.col_stop],
        alpha=alpha, beta=beta, inner_iters=inner_iters, converge_tol=converge_tol)


def divergence(bi: int, bj: int, entry: int, iteration: int) -> DivergenceError:
    return DivergenceError(
        f"block ({bi}, {bj}): non-finite residual at entry {entry}, "
        f"inner iteration {iteration}; reduce alpha",
        block=(bi, bj), entry=entry, iteration=iteration)


class _Slices:
    """Contiguous fp64 working copies of the task's slices (no copy when the
    views already are), written back after the call."""

    def __init__(self, task: BlockTask):
        self.task = task
        self.u = task.u_slice if _is_c64(task.u_slice) else np.ascontiguousarray(task.u_slice, np.float64)
        self.v = task.v_slice if _is_c64(task.v_slice) else np.ascontiguousarray(task.v_slice, np.float64)

    def write_back(self):
        if self.u is not self.task.u_slice:
            self.task.u_slice[...] = self.u
        if self.v is not self.task.v_slice:
            self.task.v_slice[...] = self.v


def _is_c64(a: np.ndarray) -> bool:
    return a.dtype == np.float64 and a.flags.c_contiguous and a.flags.writeable


def sgd_block(task: BlockTask) -> BlockStats:
    """Fixed mode: exactly inner_iters sweeps; converge mode: until the block
    RMSE improves by < converge_tol, capped at CONVERGE_CAP sweeps."""
    L = N.load()
    rows, cols, vals = N.i64(task.rows), N.i64(task.cols), N.f64(task.values)
    sl = _Slices(task)
    k = sl.u.shape[1]
    sb, sa = ctypes.c_double(), ctypes.c_double()
    be, bit = ctypes.c_int64(), ctypes.c_int64()
    if task.inner_iters is None:
        used, capped = ctypes.c_int64(), ctypes.c_int32()
        rc = L.bgmf_sgd_converge(
            N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(vals, N._f64p), len(rows),
            N.ptr(sl.u, N._f64p), sl.u.shape[0], N.ptr(sl.v, N._f64p), sl.v.shape[0], k,
            task.alpha, task.beta, task.converge_tol, CONVERGE_CAP, ctypes.byref(sb),
            ctypes.byref(sa), ctypes.byref(used), ctypes.byref(capped), ctypes.byref(be),
            ctypes.byref(bit))
        N.check(rc)
        sl.write_back()
        if be.value >= 0:
            raise divergence(task.bi, task.bj, be.value, bit.value)
        return BlockStats(sb.value, sa.value, len(rows), int(used.value), bool(capped.value))
    rc = L.bgmf_sgd_sweeps(
        N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(vals, N._f64p), len(rows),
        N.ptr(sl.u, N._f64p), sl.u.shape[0], N.ptr(sl.v, N._f64p), sl.v.shape[0], k,
        task.alpha, task.beta, int(task.inner_iters), ctypes.byref(sb), ctypes.byref(sa),
        ctypes.byref(be), ctypes.byref(bit))
    N.check(rc)
    sl.write_back()
    if be.value >= 0:
        raise divergence(task.bi, task.bj, be.value, bit.value)
    return BlockStats(sb.value, sa.value, len(rows), int(task.inner_iters))


def block_sse(task: BlockTask) -> float:
    """Squared residual sum of the task's block, no mutation (_kernels.py:16-28)."""
    L = N.load()
    rows, cols, vals = N.i64(task.rows), N.i64(task.cols), N.f64(task.values)
    u = np.ascontiguousarray(task.u_slice, np.float64)
    v = np.ascontiguousarray(task.v_slice, np.float64)
    out = ctypes.c_double()
    N.check(L.bgmf_block_sse(N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(vals, N._f64p),
                             len(rows), N.ptr(u, N._f64p), u.shape[0], N.ptr(v, N._f64p),
                             v.shape[0], u.shape[1], ctypes.byref(out)))
    return out.value


def batch_gradient_block(task: BlockTask) -> BlockStats:
    """Full-batch gradient updates on the block (kernel.py:142-158): the
    verification variant of sgd_block, through ``bgmf_gradient_steps`` (GPU,
    fp64, the reference's accumulation order: bit-identical)."""
    if task.inner_iters is None:
        raise ValueError("converge mode is only defined for sgd_block")
    L = N.load()
    rows, cols, vals = N.i64(task.rows), N.i64(task.cols), N.f64(task.values)
    sl = _Slices(task)
    sb, sa = ctypes.c_double(), ctypes.c_double()
    be, bit = ctypes.c_int64(), ctypes.c_int64()
    N.check(L.bgmf_gradient_steps(
        N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(vals, N._f64p), len(rows),
        N.ptr(sl.u, N._f64p), sl.u.shape[0], N.ptr(sl.v, N._f64p), sl.v.shape[0],
        sl.u.shape[1], task.alpha, task.beta, int(task.inner_iters), ctypes.byref(sb),
        ctypes.byref(sa), ctypes.byref(be), ctypes.byref(bit)))
    sl.write_back()
    if be.value >= 0:
        raise divergence(task.bi, task.bj, be.value, bit.value)
    return BlockStats(sb.value, sa.value, len(rows), int(task.inner_iters))


def _gradients(task: BlockTask, want_grads: bool):
    L = N.load()
    rows, cols, vals = N.i64(task.rows), N.i64(task.cols), N.f64(task.values)
    u = np.ascontiguousarray(task.u_slice, np.float64)
    v = np.ascontiguousarray(task.v_slice, np.float64)
    gu = np.empty_like(u) if want_grads else None
    gv = np.empty_like(v) if want_grads else None
    sse, reg = ctypes.c_double(), ctypes.c_double()
    N.check(L.bgmf_block_gradients(
        N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(vals, N._f64p), len(rows),
        N.ptr(u, N._f64p), u.shape[0], N.ptr(v, N._f64p), v.shape[0], u.shape[1],
        float(task.beta), None if gu is None else N.ptr(gu, N._f64p),
        None if gv is None else N.ptr(gv, N._f64p), ctypes.byref(sse), ctypes.byref(reg)))
    return sse.value + 0.5 * task.beta * reg.value, gu, gv


def block_objective(task: BlockTask) -> float:
    """Squared residual sum plus (beta/2) times the slice norms; pure
    (kernel.py:161-168).  GPU fp64."""
    return float(_gradients(task, False)[0])


def block_gradients(task: BlockTask) -> tuple[np.ndarray, np.ndarray]:
    """Analytic gradients of block_objective w.r.t. the two slices; pure
    (kernel.py:171-179).  GPU fp64, accumulated in entry order like np.add.at."""
    _, gu, gv = _gradients(task, True)
    return gu, gv
