"""paper_2304_13724_b200 -- B200-native blocked-SGD matrix factorization.

Drop-in for the BGMF hot path of the reference ``blockmf`` package
(arXiv 2304.13724): same public names, arguments, defaults and exception
types for partition / schedule / block kernel / train loop / RMSE
(reference ``pkg/src/blockmf/__init__.py:10-136``), with the numeric work in
hand-written sm_100a CUDA (``libbgmf.so``, C ABI in ``include/bgmf.h``).
There is no CPU fallback: numeric calls raise ``NativeUnavailable`` when the
library or the GPU is missing.

Also provided: the CMF / CPMF baseline trainers
(train_sequential, train_sync_parallel) and the verification kernels
(batch_gradient_block, block_objective, block_gradients) on the GPU,
sweep_budget / auto_splits over train_blocked, and the file formats and model /
trace persistence as host helpers (data.py).  Not provided: CLI and plots.
"""

from ._native import CudaError, NativeUnavailable
from .core import (AdaptiveDecreasing, Constant, ConvergeEachBlock, ConvergenceTrace,
                   DataError, Decreasing, DivergenceError, FactorModel, IncreasingEvery,
                   InnerSchedule, RatingsDataset, RatingTriple, TraceStep, TrainConfig,
                   format_schedule, init_factors, parse_schedule, validate_dataset)
from .data import (FORMATS, SyntheticSpec, gen_synthetic, load, load_model, read_trace,
                   save_dataset, save_model, split, write_trace)
from .device import Engine, EngineOptions
from .kernel import (BlockStats, BlockTask, batch_gradient_block, block_gradients,
                     block_objective, block_sse, sgd_block, task_from_block)
from .metrics import HoldoutEvaluator, RmseAccumulator, finalize, merge, rmse, test_rmse
from .partition import (Block, BlockedDataset, BlockGrid, block_dataset, locate, make_grid,
                        partition, permute_dataset, split_bounds)
from .scheduler import Batch, StepPlan, format_plan, plan_step, validate_plan
from .trainer import (SweepPoint, TrainResult, auto_splits, resolve_inner_iters, sweep_budget,
                      train_blocked)
from .baselines import train_sequential, train_sync_parallel

__all__ = [
    "FORMATS", "load", "load_model", "read_trace", "save_dataset", "save_model", "write_trace",
    "AdaptiveDecreasing", "Batch", "Block", "BlockedDataset", "BlockGrid", "BlockStats",
    "BlockTask", "Constant", "ConvergeEachBlock", "ConvergenceTrace", "CudaError", "DataError",
    "Decreasing", "DivergenceError", "Engine", "EngineOptions", "FactorModel",
    "HoldoutEvaluator", "IncreasingEvery", "InnerSchedule", "NativeUnavailable",
    "RatingTriple", "RatingsDataset", "RmseAccumulator", "StepPlan", "SyntheticSpec",
    "TraceStep", "TrainConfig", "TrainResult", "block_dataset", "block_sse", "finalize",
    "format_plan", "format_schedule", "gen_synthetic", "init_factors", "locate", "make_grid",
    "merge", "parse_schedule", "partition", "permute_dataset", "plan_step",
    "resolve_inner_iters", "rmse", "sgd_block", "split", "split_bounds", "task_from_block",
    "test_rmse", "train_blocked", "validate_dataset", "validate_plan",
    "SweepPoint", "auto_splits", "batch_gradient_block", "block_gradients", "block_objective",
    "sweep_budget", "train_sequential", "train_sync_parallel",
]

__version__ = "0.1.0"
