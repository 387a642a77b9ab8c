"""Sweep + SSE throughput of one multi-GPU rank's work on one GPU: the C4
partition trained with every stratum cut into sub-batches of `blocks` blocks
(an 8-GPU ring rank runs 2 of the 16 blocks of a stratum per batch), timed
with the engine's CUDA events.  Usage: python scripts/rank_probe.py [blocks]"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2304_13724_b200 import scheduler, workloads  # noqa: E402
from paper_2304_13724_b200.device import Engine, EngineOptions  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workloads.CONFIGS["C4"]
r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=w.seed)
eng = Engine(EngineOptions(timing=True))
eng._opt("ord_col_conc", 6.0)  # as a ring rank (distributed.GpuShard)
eng.partition(r, c, v, w.n, w.m, w.grid, w.grid)
eng.init_factors(w.n, w.m, w.k, 0)
for step in range(4):
    plan = scheduler.plan_step(w.grid, w.grid, step)
    sub = [b.blocks[i:i + per] for b in plan.batches for i in range(0, len(b.blocks), per)]
    ids, off = eng.plan_arrays(sub)
    if step == 1:
        eng.kernel_stats(reset=True)
    sse, bad = eng.run_step(ids, off, 1, w.alpha, w.beta)[:2]
st = eng.kernel_stats()
# host enqueue cost of a ring rank: step_begin / step_batch per batch / step_end,
# while the GPU runs (what each of 8 ranks pays per stratum on its own host thread)
import time  # noqa: E402
plan = scheduler.plan_step(w.grid, w.grid, 0)
sub = [b.blocks[i:i + per] for b in plan.batches for i in range(0, len(b.blocks), per)]
arrs = [eng.plan_arrays([bl]) for bl in sub]
eng.step_begin(len(sub) * per)
t0 = time.perf_counter()
for ids, off in arrs:
    eng.step_batch(ids, off, 1, w.alpha, w.beta)
t_enq = time.perf_counter() - t0
eng.step_end()
print(f"host enqueue: {1e6 * t_enq / len(arrs):.1f} us per batch of {per} blocks "
      f"(step_batch: work table + sweep + SSE launches)", flush=True)
n3 = 3 * w.nnz
print(f"blocks/launch={per}: sweep {st['sgd_ms'] / 3:.3f} ms/epoch "
      f"({n3 / st['sgd_ms'] / 1e6:.2f} G/s), SSE {st['sse_ms'] / 3:.3f} ms/epoch, "
      f"epoch {n3 / (st['sgd_ms'] + st['sse_ms']) / 1e6:.2f} G upd/s, "
      f"{st['sgd_launches'] // 3} sweep launches/epoch; "
      f"train rmse {np.sqrt(sse.sum() / w.nnz):.6f}", flush=True)
eng.close()
