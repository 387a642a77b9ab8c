"""One rank of the GPU ring trainer for tests/test_gpu_ring_multirank.py:
several ranks share ONE GPU over gloo (BGMF_DIST_BACKEND=gloo, BGMF_DEVICE=0;
V moves and collectives staged through host memory).  Launched by torchrun;
rank 0 writes the trace and a model digest as JSON to argv[1]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from paper_2304_13724_b200 import distributed as D  # noqa: E402
from paper_2304_13724_b200 import workloads  # noqa: E402


def main(out_path: str, case: str) -> None:
    r, c, v = workloads.lowrank(6040, 3706, 300_000, seed=11)
    d = bm.RatingsDataset(6040, 3706, r, c, v)
    test = None
    if case == "holdout":
        d, test = bm.split(d, 0.2, seed=3)
    if case.startswith("diverge"):  # every rank must raise the same step
        cfg = bm.TrainConfig(k=32, outer_steps=3, grid_i=8, grid_j=8, alpha=1e9)
        try:
            D.train_blocked_distributed(d, cfg, early_stop=case.endswith("es"))
            err = None
        except bm.DivergenceError as e:
            err = {"step": e.step, "block": list(e.block) if e.block else None,
                   "partial": len(e.partial_trace)}
        json.dump(err, open(f"{out_path}.{os.environ['RANK']}", "w"))
        return
    sched = {"const": bm.Constant(1), "inc": bm.IncreasingEvery(2, 3),
             "converge": bm.ConvergeEachBlock(0.5), "holdout": bm.Constant(1),
             "stream": bm.Constant(1), "stream_inc": bm.IncreasingEvery(2, 3)}[case]
    cfg = bm.TrainConfig(k=32, outer_steps=4, grid_i=8, grid_j=8, inner_schedule=sched)
    # "stream*": every rank out of core -- its row shard partitioned in chunks
    # under a device budget of ~40k ratings into pinned memory, streamed
    # through a 3-slot ring inside the asynchronous ring steps
    opts = (bm.EngineOptions(device_rating_budget=12 * 40_000, stream_slots=3)
            if case.startswith("stream") else None)
    model, trace, stop = D.train_blocked_distributed(d, cfg, test, early_stop=False,
                                                     options=opts)
    if int(os.environ["RANK"]) == 0:
        json.dump({"train": [s.train_rmse for s in trace],
                   "test": [s.test_rmse for s in trace],
                   "iters": [s.inner_iters for s in trace],
                   "stop": stop, "u_shape": list(model.u.shape),
                   "rmse": bm.rmse(model, d), "finite": bool(np.isfinite(model.u).all()
                                                             and np.isfinite(model.v).all())},
                  open(out_path, "w"))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
