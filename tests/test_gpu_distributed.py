"""The NCCL multi-GPU trainer on the one GPU this run has: world_size 1
exercises GpuShard (torch-allocated U/V bound into the engine), the ring
schedule, NCCL all-reduce of the per-block SSEs and the final gather; the
trace must match the oracle per epoch (1e-3) like the single-GPU trainer.
Multi-rank routing of V blocks is covered on CPU/gloo by
test_distributed_cpu.py."""

import os
import socket

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from oracle import oracle as O
from paper_2304_13724_b200 import workloads

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world1_nccl_matches_oracle():
    import torch.distributed as dist

    from paper_2304_13724_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        r, c, v = workloads.lowrank(6040, 3706, 500_000, seed=5)
        d, te = bm.split(bm.RatingsDataset(6040, 3706, r, c, v), 0.2, seed=1)
        cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8)
        model, trace, stop = D.train_blocked_distributed(d, cfg, te, early_stop=False)
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=4,
                                       grid_i=8, grid_j=8, early_stop=False, nthreads=8,
                                       test=(te.rows, te.cols, te.values))
        got = np.array([s.train_rmse for s in trace])
        assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= 1e-3
        got_t = np.array([s.test_rmse for s in trace])
        assert np.abs(got_t - [s["test_rmse"] for s in otr]).max() <= 1e-3
        assert stop == "max_steps" and model.u.shape == (6040, 32)
        assert np.isfinite(bm.rmse(model, d))
    finally:
        dist.destroy_process_group()


def test_async_step_matches_run_step():
    """bgmf_step_begin/_batch/_end (the ring trainer's per-stratum path) gives
    the same per-block SSEs as one bgmf_run_step over the whole plan, and
    reports divergence by block id in submission order."""
    r, c, v = workloads.lowrank(6040, 3706, 400_000, seed=9)
    P = 4
    plan = bm.plan_step(P, P, 0)
    outs = []
    for mode in ("sync", "async"):
        eng = bm.Engine()
        eng.partition(r, c, v, 6040, 3706, P, P)
        eng.init_factors(6040, 3706, 32, 0)
        if mode == "sync":
            ids, off = eng.plan_arrays(plan)
            sse, bad = eng.run_step(ids, off, 1, 1e-3, 1e-2)
        else:
            eng.step_begin(P * P)
            for batch in plan:
                ids, off = eng.plan_arrays([batch])
                eng.step_batch(ids, off, 1, 1e-3, 1e-2)
            sse, bad = eng.step_end()
        assert bad is None
        outs.append(sse)
        eng.close()
    np.testing.assert_allclose(outs[1], outs[0], rtol=1e-5)
    eng = bm.Engine()
    eng.partition(r, c, v, 6040, 3706, P, P)
    eng.init_factors(6040, 3706, 32, 0)
    eng.step_begin(P * P)
    for batch in plan:
        ids, off = eng.plan_arrays([batch])
        eng.step_batch(ids, off, 1, 1e9, 0.0)
    sse, bad = eng.step_end()
    first = plan.batches[0].blocks[0]
    assert bad is not None and bad[0] == first[0] * P + first[1]
    with pytest.raises(RuntimeError, match="step_begin"):
        eng.step_batch(ids, off, 1, 1e-3, 1e-2)  # no step_begin


def test_world1_nccl_adaptive_schedule_matches_oracle():
    """AdaptiveDecreasing in the ring trainer: the inner-iteration count
    follows the improvement ratio of the global trace (trainer.py:52-73)."""
    import torch.distributed as dist

    from paper_2304_13724_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        r, c, v = workloads.lowrank(6040, 3706, 300_000, seed=7)
        d = bm.RatingsDataset(6040, 3706, r, c, v)
        cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8, alpha=1e-3,
                             inner_schedule=bm.AdaptiveDecreasing(4))
        _, trace, _ = D.train_blocked_distributed(d, cfg, early_stop=False)
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=4,
                                       alpha=1e-3, grid_i=8, grid_j=8, schedule="adaptive:4",
                                       early_stop=False, nthreads=8)
        assert [s.inner_iters for s in trace] == [s["inner_iters"] for s in otr]
        got = np.array([s.train_rmse for s in trace])
        assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= 1e-3
    finally:
        dist.destroy_process_group()


def test_world1_nccl_converge_schedule_matches_oracle():
    """ConvergeEachBlock in the ring trainer: per-block sweep counts and
    capped blocks reduced over the ranks, trace within 1e-3 of the oracle."""
    import torch.distributed as dist

    from paper_2304_13724_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        d = bm.gen_synthetic(bm.SyntheticSpec(64, 64, 1, 30, seed=0))
        cfg = bm.TrainConfig(k=10, outer_steps=2, grid_i=4, grid_j=4,
                             inner_schedule=bm.ConvergeEachBlock(0.5))
        _, trace, _ = D.train_blocked_distributed(d, cfg, early_stop=False,
                                                  options=bm.EngineOptions(min_chunk=1 << 20))
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=10, outer_steps=2,
                                       grid_i=4, grid_j=4, schedule="converge:0.5",
                                       early_stop=False)
        got = np.array([s.train_rmse for s in trace])
        assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= 1e-3
        assert all(s.inner_iters >= 1 for s in trace)
    finally:
        dist.destroy_process_group()


def test_gpu_shard_refuses_the_legacy_default_stream():
    """The ring's ordering (sweep -> NCCL send of its V block -> recv -> next
    sweep) holds only if the engine, NCCL and torch share one stream; on the
    legacy default stream the engine would run on a private stream."""
    import torch
    import torch.distributed as dist

    from paper_2304_13724_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        d = bm.gen_synthetic(bm.SyntheticSpec(64, 64, 1, 30, seed=0))
        cfg = bm.TrainConfig(k=8, outer_steps=1, grid_i=4, grid_j=4)
        sched = D.RingSchedule(4, 4, 1)
        with torch.cuda.stream(torch.cuda.default_stream(0)):
            with pytest.raises(RuntimeError, match="non-default"):
                D.GpuShard(d, cfg, sched, 0, 0)
        s = torch.cuda.Stream(0)
        with torch.cuda.stream(s):
            shard = D.GpuShard(d, cfg, sched, 0, 0)
            assert shard.stream.cuda_stream == s.cuda_stream
            shard.eng.close()
    finally:
        dist.destroy_process_group()


def test_world1_nccl_batched_epochs_match_oracle_and_divergence():
    """Fixed schedule, no early stop, no holdout: the epochs run back to back
    with device-resident SSEs (bgmf_step_end_async); trace within 1e-3 of the
    oracle, per-step seconds from CUDA events.  A diverging run raises the
    same DivergenceError (step, block) batched and per step."""
    import torch.distributed as dist

    from paper_2304_13724_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        r, c, v = workloads.lowrank(6040, 3706, 400_000, seed=7)
        d = bm.RatingsDataset(6040, 3706, r, c, v)
        cfg = bm.TrainConfig(k=32, outer_steps=5, grid_i=8, grid_j=8,
                             inner_schedule=bm.IncreasingEvery(2, 3))
        model, trace, stop = D.train_blocked_distributed(d, cfg, early_stop=False)
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=5,
                                       grid_i=8, grid_j=8, early_stop=False, nthreads=8,
                                       schedule="inc:2,3")
        got = np.array([s.train_rmse for s in trace])
        assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= 1e-3
        assert [s.inner_iters for s in trace] == [s["inner_iters"] for s in otr]
        assert all(s.seconds > 0 for s in trace) and stop == "max_steps"
        bad = bm.TrainConfig(k=32, outer_steps=3, grid_i=8, grid_j=8, alpha=1e9)
        errs = []
        for es in (False, True):  # batched, then per step
            with pytest.raises(bm.DivergenceError) as ei:
                D.train_blocked_distributed(d, bad, early_stop=es)
            errs.append((ei.value.step, ei.value.block))
        assert errs[0] == errs[1] and errs[0][0] == 1
    finally:
        dist.destroy_process_group()
