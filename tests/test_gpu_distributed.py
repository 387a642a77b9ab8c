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
        d = bm.RatingsDataset(6040, 3706, r, c, v)
        cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8)
        model, trace, stop = D.train_blocked_distributed(d, cfg, early_stop=False)
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=32, outer_steps=4,
                                       grid_i=8, grid_j=8, early_stop=False, nthreads=8)
        got = np.array([s.train_rmse for s in trace])
        assert np.abs(got - [s["train_rmse"] for s in otr]).max() <= 1e-3
        assert stop == "max_steps" and model.u.shape == (6040, 32)
        assert np.isfinite(bm.rmse(model, d))
    finally:
        dist.destroy_process_group()
