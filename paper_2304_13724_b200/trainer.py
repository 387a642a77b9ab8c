"""Blocked training loop on the GPU (reference ``trainer.py:38-184``).

The host keeps only what is O(steps) or O(P^2): schedule resolution,
``plan_step``, the merge of per-block SSEs in submission order, the trace and
early stopping.  Each outer step is ONE ``bgmf_run_step`` call: every stratum
of the plan runs as a kernel launch over all of its blocks at once (plus the
post-sweep SSE launch the trace needs), ratings and factors never leave HBM,
and only the P^2 per-block SSEs come back.
"""

from __future__ import annotations

import math
import os
import sys
import time
from dataclasses import dataclass
from typing import Callable, Literal, Optional

import numpy as np

from .core import (AdaptiveDecreasing, Constant, ConvergeEachBlock, ConvergenceTrace,
                   Decreasing, DivergenceError, FactorModel, IncreasingEvery, InnerSchedule,
                   RatingsDataset, TraceStep, TrainConfig, init_factors)
from .device import EngineOptions
from .kernel import CONVERGE_CAP, BlockTask, divergence
from .metrics import HoldoutEvaluator, RmseAccumulator, finalize, merge
from .partition import BlockedDataset, make_grid
from .scheduler import plan_step

StopReason = Literal["converged", "max_steps", "diverged"]
BlockHook = Callable[[str, BlockTask], None]


@dataclass(frozen=True)
class TrainResult:
    model: FactorModel
    trace: ConvergenceTrace
    stop_reason: StopReason


def resolve_inner_iters(schedule: InnerSchedule, step: int,
                        prev_improvement_ratio: float = 1.0) -> Optional[int]:
    """Sweeps for 1-based outer step ``step`` (trainer.py:52-73); None means
    converge-each-block."""
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    if isinstance(schedule, Constant):
        return schedule.iters
    if isinstance(schedule, IncreasingEvery):
        return min(math.ceil(step / schedule.period), schedule.cap)
    if isinstance(schedule, Decreasing):
        return max(schedule.start - step + 1, 1)
    if isinstance(schedule, AdaptiveDecreasing):
        return max(round(schedule.start * prev_improvement_ratio), 1)
    if isinstance(schedule, ConvergeEachBlock):
        return None
    raise TypeError(f"not a schedule: {schedule!r}")


class _HookTasks:
    """BlockTask objects handed to ``block_hook``.  Entry arrays are the
    block's host views; factor slices are views of a host mirror of the
    initial factors (the live factors are in HBM)."""

    def __init__(self, blocked: BlockedDataset, model: FactorModel, cfg: TrainConfig):
        self.blocked, self.model, self.cfg = blocked, model, cfg

    def make(self, bi: int, bj: int, g, tol) -> BlockTask:
        b = self.blocked.block(bi, bj)
        return BlockTask(bi=bi, bj=bj, rows=b.rows, cols=b.cols, values=b.values,
                         u_slice=self.model.u[b.row_start:b.row_stop],
                         v_slice=self.model.v[b.col_start:b.col_stop],
                         alpha=self.cfg.alpha, beta=self.cfg.beta,
                         inner_iters=g, converge_tol=tol if g is None else 0.0)


def train_blocked(d: RatingsDataset, cfg: TrainConfig, test: Optional[RatingsDataset] = None,
                  *, early_stop: bool = True, timing: bool = True,
                  block_hook: Optional[BlockHook] = None,
                  options: Optional[EngineOptions] = None,
                  blocked: Optional[BlockedDataset] = None) -> TrainResult:
    """Blocked SGD factorization of ``d`` (same contract as trainer.py:76-184).

    B200 additions (keyword-only, optional): ``options`` selects the engine
    (fast fp32 lossless kernels by default, ``EngineOptions(exact=True)`` for
    the fp64 bit-exact kernels); ``blocked`` reuses an existing GPU partition
    of ``d`` with the same grid.  ``cfg.workers`` is ignored: concurrency is
    the GPU's.
    """
    prof = _Phases() if os.environ.get("BGMF_PROFILE") else None
    own = blocked is None
    if own:
        blocked = BlockedDataset(d, make_grid(d.n, d.m, cfg.grid_i, cfg.grid_j), options)
    if prof:
        prof.mark("partition (H2D + GPU sort)")
    if (blocked.grid.grid_i, blocked.grid.grid_j) != (cfg.grid_i, cfg.grid_j) \
            or blocked.dataset is not d:
        raise ValueError("blocked must partition d with cfg's grid")
    try:
        eng = blocked.engine
        # init_factors(n, m, k, seed) generated in HBM: numpy's PCG64 stream
        # reproduced bit-for-bit on the device (no 2*(n+m)*k*8-byte upload)
        eng.init_factors(d.n, d.m, cfg.k, cfg.seed)
        if prof:
            prof.mark("init_factors (device PCG64)")

        evaluator = HoldoutEvaluator(d, test) if test is not None and len(test) > 0 else None
        if evaluator is not None:
            t = evaluator.test
            eng.holdout_set(t.rows, t.cols, t.values, evaluator.cold, evaluator.fallback)
        sched = cfg.inner_schedule
        tol = sched.tol if isinstance(sched, ConvergeEachBlock) else 0.0
        adaptive = isinstance(sched, AdaptiveDecreasing)
        hist = [math.sqrt(eng.train_sse() / len(d))] if adaptive and len(d) else [0.0]
        counts = np.diff(eng.offsets)
        hooks = (_HookTasks(blocked, init_factors(d.n, d.m, cfg.k, cfg.seed), cfg)
                 if block_hook is not None else None)

        trace = ConvergenceTrace()
        stop: StopReason = "max_steps"
        batched = (not early_stop and block_hook is None and evaluator is None and not adaptive
                   and not isinstance(sched, ConvergeEachBlock) and not eng.options.exact
                   and not eng.streaming and cfg.outer_steps > 1)
        if own:  # fault the model's output pages in while the epochs run
            eng.prefault_factors()
        if batched:
            # nothing is decided on the host between steps: enqueue every epoch
            # in one bgmf_run_steps call (no host round trip between epochs)
            _run_steps_batched(eng, cfg, sched, counts, trace, timing)
        for step in range(1, 0 if batched else cfg.outer_steps + 1):
            if adaptive and step >= 2:
                prev, cur = hist[-2], hist[-1]
                ratio = (prev - cur) / prev if prev > 0 else 0.0
            else:
                ratio = 1.0
            g = resolve_inner_iters(sched, step, ratio)
            t0 = time.perf_counter()
            batches = plan_step(cfg.grid_i, cfg.grid_j, step - 1)
            try:
                acc, max_iters, capped = _run_step(eng, batches, g, tol, cfg, counts, hooks,
                                                   block_hook)
            except DivergenceError as exc:
                exc.step = step
                exc.partial_trace = trace
                raise
            train_rmse = finalize(acc)
            test_rmse = (math.sqrt(eng.holdout_sse() / len(evaluator.test))
                         if evaluator is not None else None)
            trace.append(TraceStep(step=step, train_rmse=train_rmse, test_rmse=test_rmse,
                                   seconds=time.perf_counter() - t0 if timing else 0.0,
                                   inner_iters=max_iters, capped_blocks=capped))
            hist.append(train_rmse)
            if early_stop:
                if acc.count == 0:
                    stop = "converged"
                    break
                if len(trace) >= 2 and trace.steps[-2].train_rmse - train_rmse < cfg.delta:
                    stop = "converged"
                    break
        if prof:
            prof.mark(f"{len(trace)} epochs")
        u, v = eng.get_factors()
        if prof:
            prof.mark("get_factors (D2H)")
        if own:  # the partition was made for this call: release its HBM now
            eng.close()
        if prof:
            prof.mark("release device context")
            prof.report()
        return TrainResult(model=FactorModel(u, v), trace=trace, stop_reason=stop)
    except BaseException:
        if own:  # a failed call (DivergenceError, interrupt) releases its HBM too
            blocked.engine.close()
        raise


class _Phases:
    """BGMF_PROFILE=1: wall time of train_blocked's phases on stderr."""

    def __init__(self):
        self.t = time.perf_counter()
        self.rows = []

    def mark(self, what):
        now = time.perf_counter()
        self.rows.append((what, now - self.t))
        self.t = now

    def report(self):
        for what, dt in self.rows:
            print(f"[bgmf] {what:32s} {dt * 1e3:9.2f} ms", file=sys.stderr)


def _run_steps_batched(eng, cfg, sched, counts, trace, timing):
    """All outer steps of a fixed-schedule, no-early-stop run in one engine
    call; the trace (and a DivergenceError at the first diverged step, with
    the trace before it) as the per-step loop would produce."""
    steps = []
    for step in range(1, cfg.outer_steps + 1):
        g = resolve_inner_iters(sched, step, 1.0)
        ids, off = eng.plan_arrays(plan_step(cfg.grid_i, cfg.grid_j, step - 1))
        steps.append((ids, off, g))
    sse_all, bad, ms = eng.run_steps(steps, cfg.alpha, cfg.beta)
    for k, (ids, _, g) in enumerate(steps):
        sse = sse_all[k]
        pos_bad, entry, it = None, None, None
        if bad is not None and bad[0] == k:
            pos_bad = int(np.nonzero(ids == bad[1])[0][0])
            entry, it = bad[2], bad[3]
        # the reference also stops at a non-finite post-sweep SSE
        # (_kernels.py:57-58); the first offender in plan order wins
        for pos, b in enumerate(ids):
            if pos_bad is not None and pos >= pos_bad:
                break
            if not math.isfinite(sse[b]):
                pos_bad, entry, it = pos, int(counts[b]) - 1, g - 1
                break
        if pos_bad is not None:
            b = int(ids[pos_bad])
            exc = divergence(b // cfg.grid_j, b % cfg.grid_j, entry, it)
            exc.step = k + 1
            exc.partial_trace = trace
            raise exc
        acc = RmseAccumulator()
        for b in ids:  # submission order, as trainer.py:149-152
            acc = merge(acc, RmseAccumulator(float(sse[b]), int(counts[b])))
        trace.append(TraceStep(step=k + 1, train_rmse=finalize(acc), test_rmse=None,
                               seconds=float(ms[k]) / 1e3 if timing else 0.0, inner_iters=g,
                               capped_blocks=0))


def _run_step(eng, batches, g, tol, cfg, counts, hooks, block_hook):
    """One outer step; returns (accumulator, max inner iters, capped blocks)."""
    acc = RmseAccumulator()
    max_iters, capped = 0, 0
    # with a hook, launch batch by batch so "start"/"end" bracket each stratum
    groups = [[b] for b in batches] if block_hook is not None else [list(batches)]
    for group in groups:
        ids, off = eng.plan_arrays(group)
        tasks = []
        if block_hook is not None:
            tasks = [hooks.make(bi, bj, g, tol) for bi, bj in group[0]]
            for t in tasks:
                block_hook("start", t)
        try:
            if g is None:
                sse, iters, cap, bad = eng.run_step_converge(ids, off, tol, CONVERGE_CAP,
                                                             cfg.alpha, cfg.beta)
            else:
                sse, bad = eng.run_step(ids, off, g, cfg.alpha, cfg.beta)
        finally:
            for t in tasks:
                block_hook("end", t)
        # the reference also stops at a non-finite post-sweep SSE
        # (_kernels.py:57-58); the first offender in plan order wins
        for pos, b in enumerate(ids):
            if bad is not None and pos >= bad[0]:
                break
            if not math.isfinite(sse[b]):
                last_it = (g if g is not None else max(int(iters[b]), 1)) - 1
                bad = (pos, int(counts[b]) - 1, last_it)
                break
        if bad is not None:
            pos, entry, it = bad
            b = int(ids[pos])
            raise divergence(b // cfg.grid_j, b % cfg.grid_j, entry, it)
        for b in ids:  # submission order, as trainer.py:149-152
            acc = merge(acc, RmseAccumulator(float(sse[b]), int(counts[b])))
            if g is None:
                max_iters = max(max_iters, int(iters[b]))
                capped += int(cap[b])
        if g is not None:
            max_iters = g
    return acc, max_iters, capped


@dataclass(frozen=True)
class SweepPoint:
    """Outcome of one (outer, inner) split of a fixed iteration budget
    (trainer.py:187-194)."""

    outer: int
    inner: int
    final_rmse: float
    seconds: float


def auto_splits(total_budget: int) -> list[tuple[int, int]]:
    """All (outer, inner) factorizations of the budget, ascending outer
    (trainer.py:197-205)."""
    if total_budget < 1:
        raise ValueError(f"budget must be >= 1, got {total_budget}")
    return [(outer, total_budget // outer) for outer in range(1, total_budget + 1)
            if total_budget % outer == 0]


def sweep_budget(d: RatingsDataset, cfg: TrainConfig, total_budget: int,
                 splits: list[tuple[int, int]], *, timing: bool = True,
                 options: Optional[EngineOptions] = None) -> list[SweepPoint]:
    """One training run per (outer, inner) split of a fixed total iteration
    budget, Constant(inner) for exactly ``outer`` steps from the same seeded
    init (trainer.py:208-248).  final_rmse is the full-dataset RMSE of the
    finished model (GPU), not the trace value.  The partition is built once
    and reused by every split."""
    from dataclasses import replace

    from .metrics import rmse

    for outer, inner in splits:
        if outer < 1 or inner < 1 or outer * inner != total_budget:
            raise ValueError(f"split ({outer}, {inner}) does not factor budget {total_budget}")
    points = []
    blocked = None
    try:
        for outer, inner in splits:
            if blocked is None and len(splits) > 1:
                blocked = BlockedDataset(d, make_grid(d.n, d.m, cfg.grid_i, cfg.grid_j), options)
            run_cfg = replace(cfg, outer_steps=outer, inner_schedule=Constant(inner))
            t0 = time.perf_counter()
            result = train_blocked(d, run_cfg, early_stop=False, timing=timing, options=options,
                                   blocked=blocked)
            seconds = time.perf_counter() - t0 if timing else 0.0
            points.append(SweepPoint(outer=outer, inner=inner,
                                     final_rmse=rmse(result.model, d), seconds=seconds))
    finally:
        if blocked is not None:
            blocked.engine.close()
    return points
