"""Baseline trainers on the GPU (reference ``baselines.py``).

* :func:`train_sequential` (CMF, baselines.py:62-97) is plain SGD, one
  row-major pass over all entries per outer step -- by the reference's own
  contract bit-identical to ``train_blocked`` with a 1x1 grid and Constant(1)
  (test_trainer.py:33-41), which is how it runs here.
* :func:`train_sync_parallel` (CPMF, baselines.py:100-182) splits the
  row-major entries into ``cfg.workers`` contiguous row shards; per outer step
  every shard sweeps once, updating U in place and a private copy of V, then
  the V deltas are summed in shard order.  One ``bgmf_run_sync_parallel_step``
  per outer step runs all shards at once on the device (exact mode:
  bit-identical; fast mode: each shard chunked over worker groups).

Both take the same extra keyword as ``train_blocked``: ``options``
(:class:`EngineOptions`).
"""

from __future__ import annotations

import math
import time
from dataclasses import replace
from typing import Optional

import numpy as np

from .core import (Constant, ConvergenceTrace, DivergenceError, RatingsDataset, TraceStep,
                   TrainConfig)
from .device import EngineOptions
from .metrics import HoldoutEvaluator
from .partition import BlockedDataset, make_grid, split_bounds
from .trainer import StopReason, TrainResult, train_blocked


def train_sequential(d: RatingsDataset, cfg: TrainConfig,
                     test: Optional[RatingsDataset] = None, *, early_stop: bool = True,
                     timing: bool = True,
                     options: Optional[EngineOptions] = None) -> TrainResult:
    """Plain SGD: one row-major pass over all entries per outer step.  Grid,
    schedule and worker fields of cfg are ignored (baselines.py:62-97)."""
    cfg1 = replace(cfg, grid_i=1, grid_j=1, inner_schedule=Constant(1))
    return train_blocked(d, cfg1, test, early_stop=early_stop, timing=timing, options=options)


def _should_stop(trace: ConvergenceTrace, count: int, delta: float) -> bool:
    """baselines.py:53-58."""
    if count == 0:
        return True
    if len(trace) < 2:
        return False
    return trace.steps[-2].train_rmse - trace.steps[-1].train_rmse < delta


def train_sync_parallel(d: RatingsDataset, cfg: TrainConfig,
                        test: Optional[RatingsDataset] = None, *, early_stop: bool = True,
                        timing: bool = True,
                        options: Optional[EngineOptions] = None) -> TrainResult:
    """Row-sharded SGD with a synchronization barrier after every sweep
    (baselines.py:100-182).  Deterministic for a fixed shard count."""
    from .core import FactorModel

    blocked = BlockedDataset(d, make_grid(d.n, d.m, 1, 1), options)
    eng = blocked.engine
    try:
        eng.init_factors(d.n, d.m, cfg.k, cfg.seed)
        evaluator = HoldoutEvaluator(d, test) if test is not None and len(test) > 0 else None
        if evaluator is not None:
            t = evaluator.test
            eng.holdout_set(t.rows, t.cols, t.values, evaluator.cold, evaluator.fallback)
        shards = min(cfg.workers, max(d.n, 1))
        # entries are row-major, so shard w is one contiguous range:
        # searchsorted(rows, split_bounds(n, shards)) of baselines.py:129
        per_row = np.bincount(np.asarray(d.rows, np.int64), minlength=d.n) if len(d) else \
            np.zeros(d.n, np.int64)
        starts = np.concatenate([[0], np.cumsum(per_row)])
        edges = starts[np.asarray(split_bounds(d.n, shards), np.int64)]
        trace = ConvergenceTrace()
        stop: StopReason = "max_steps"
        for step in range(1, cfg.outer_steps + 1):
            t0 = time.perf_counter()
            sse_w, bad = eng.run_sync_parallel_step(edges, cfg.alpha, cfg.beta)
            if bad is not None:
                w, entry, it = bad
                exc = DivergenceError(
                    f"shard {w}: non-finite residual at entry {entry}; reduce alpha",
                    entry=int(entry), iteration=int(it))
                exc.step = step
                exc.partial_trace = trace
                raise exc
            sse = sum(float(x) for x in sse_w)
            count = int(edges[-1] - edges[0])
            train_rmse = float(math.sqrt(sse / count)) if count else 0.0
            test_rmse = (math.sqrt(eng.holdout_sse() / len(evaluator.test))
                         if evaluator is not None else None)
            trace.append(TraceStep(step=step, train_rmse=train_rmse, test_rmse=test_rmse,
                                   seconds=time.perf_counter() - t0 if timing else 0.0,
                                   inner_iters=1))
            if early_stop and _should_stop(trace, count, cfg.delta):
                stop = "converged"
                break
        u, v = eng.get_factors()
    finally:
        eng.close()
    return TrainResult(model=FactorModel(u, v), trace=trace, stop_reason=stop)
