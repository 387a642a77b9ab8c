"""Epoch throughput of the fast path across latent sizes k on the C4 shape
(480k x 17.8k, 100 M ratings, 16x16): sweep and SSE per epoch from the
engine's CUDA events, and the sweep's bytes/s against its algorithmic
12 + 16k B per rating.  Usage: python scripts/k_sweep.py [k ...]"""
import sys

sys.path.insert(0, ".")
from paper_2304_13724_b200 import scheduler, workloads  # noqa: E402
from paper_2304_13724_b200.device import Engine, EngineOptions  # noqa: E402

ks = [int(x) for x in sys.argv[1:]] or [16, 32, 64, 96, 128, 192, 256]
w = workloads.CONFIGS["C4"]
r, c, v = workloads.lowrank(w.n, w.m, w.nnz, seed=w.seed)
eng = Engine(EngineOptions(timing=True))
eng.partition(r, c, v, w.n, w.m, w.grid, w.grid)
for k in ks:
    eng.init_factors(w.n, w.m, k, 0)
    for step in range(5):
        ids, off = eng.plan_arrays(scheduler.plan_step(w.grid, w.grid, step).batches)
        if step == 2:
            eng.kernel_stats(reset=True)
        eng.run_step(ids, off, 1, w.alpha, w.beta)
    st = eng.kernel_stats()
    sgd, sse = st["sgd_ms"] / 3, st["sse_ms"] / 3
    print(f"k={k:4d}: sweep {sgd:7.3f} ms ({w.nnz / sgd / 1e6:6.2f} G ratings/s, "
          f"{w.nnz * (12 + 16 * k) / sgd / 1e6:7.0f} GB/s alg), SSE {sse:6.3f} ms, "
          f"epoch {w.nnz / (sgd + sse) / 1e6:5.2f} G upd/s", flush=True)
eng.close()
