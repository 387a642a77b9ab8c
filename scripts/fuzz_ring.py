"""Randomised parity of the multi-rank ring on ONE GPU (ranks share the
device over gloo; V moves over the peer transport): random world sizes,
shapes, grids, k, schedules, holdouts and out-of-core ranks (a device
budget that makes every rank stream its shard), each launched with torchrun
and compared with the oracle's single-process trace.
Usage: python scripts/fuzz_ring.py [cases] [seed]"""
import json
import os
import socket
import subprocess
import sys
import tempfile

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2304_13724_b200 as bm  # noqa: E402
from oracle import oracle as O  # noqa: E402

WORKER = r'''
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import distributed as D
spec = json.load(open(sys.argv[1]))
z = np.load(spec["data"])
d = bm.RatingsDataset(spec["n"], spec["m"], z["r"], z["c"], z["v"])
test = None
if spec["holdout"]:
    d, test = bm.split(d, 0.2, seed=1)
sched = {"const": bm.Constant(1), "inc": bm.IncreasingEvery(2, 3), "dec": bm.Decreasing(3),
         "adaptive": bm.AdaptiveDecreasing(2), "converge": bm.ConvergeEachBlock(0.05)}[spec["sched"]]
cfg = bm.TrainConfig(k=spec["k"], outer_steps=spec["steps"], grid_i=spec["I"], grid_j=spec["J"],
                     alpha=3e-4, inner_schedule=sched)
opts = (bm.EngineOptions(device_rating_budget=spec["budget"], stream_slots=3)
        if spec["budget"] else None)
try:
    model, trace, stop = D.train_blocked_distributed(d, cfg, test, early_stop=False,
                                                     options=opts)
except Exception as e:  # a slot smaller than the largest block: skip the case
    if spec["budget"] and "slot" in str(e):
        if os.environ["RANK"] == "0":
            json.dump({"skip": True}, open(spec["out"], "w"))
        sys.exit(0)
    raise
if os.environ["RANK"] == "0":
    json.dump({"train": [s.train_rmse for s in trace], "test": [s.test_rmse for s in trace]},
              open(spec["out"], "w"))
'''
SPECS = {"const": "const:1", "inc": "inc:2,3", "dec": "dec:3", "adaptive": "adaptive:2",
         "converge": "converge:0.05"}


def port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


cases = int(sys.argv[1]) if len(sys.argv) > 1 else 10
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
tmp = tempfile.mkdtemp()
open(os.path.join(tmp, "w.py"), "w").write(WORKER)
fails = 0
for i in range(cases):
    world = int(g.integers(2, 5))
    n, m = int(g.integers(world * 4, 4000)), int(g.integers(8, 4000))
    nnz = int(min(n * m, g.integers(500, 120_000)))
    cells = g.choice(n * m, nnz, replace=False)
    r, c = np.divmod(cells, m)
    v = np.clip(np.rint(3 + g.normal(0, 1, nnz)), 1, 5)
    I = int(g.integers(world, min(n, 16) + 1))
    J = int(g.integers(1, min(m, 16) + 1))
    spec = dict(n=n, m=m, k=int(g.choice([8, 16, 30, 32, 64, 96, 128])), I=I, J=J,
                steps=int(g.integers(1, 4)), sched=str(g.choice(list(SPECS))),
                holdout=bool(g.random() < 0.3), data=os.path.join(tmp, f"d{i}.npz"),
                out=os.path.join(tmp, f"o{i}.json"),
                budget=(36 * (3 * nnz // (I * J) + 64)) if g.random() < 0.35 else 0)
    np.savez(spec["data"], r=r, c=c, v=v)
    json.dump(spec, open(os.path.join(tmp, f"s{i}.json"), "w"))
    tag = f"case {i}: world={world} " + " ".join(f"{k}={spec[k]}" for k in
                                                  ("n", "m", "k", "I", "J", "steps", "sched",
                                                   "holdout", "budget")) + f" nnz={nnz}"
    env = dict(os.environ, BGMF_DIST_BACKEND="gloo", BGMF_DEVICE="0")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={port()}", os.path.join(tmp, "w.py"),
                        os.path.join(tmp, f"s{i}.json")], env=env, capture_output=True,
                       text=True, timeout=600)
    try:
        assert p.returncode == 0, p.stderr[-1500:]
        got = json.load(open(spec["out"]))
        if got.get("skip"):
            print(f"skip {tag}", flush=True)
            continue
        d = bm.RatingsDataset(n, m, r, c, v)
        test = None
        if spec["holdout"]:
            d, te = bm.split(d, 0.2, seed=1)
            test = (te.rows, te.cols, te.values)
        _, _, otr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=spec["k"],
                                       outer_steps=spec["steps"], grid_i=I, grid_j=J,
                                       alpha=3e-4, schedule=SPECS[spec["sched"]],
                                       early_stop=False, test=test)
        dtr = np.abs(np.array(got["train"]) - [s["train_rmse"] for s in otr]).max()
        assert dtr <= 1e-3, dtr
        if spec["holdout"]:
            dte = np.abs(np.array(got["test"]) - [s["test_rmse"] for s in otr]).max()
            assert dte <= 1e-3, dte
        print(f"ok   {tag}  max|d train| {dtr:.1e}", flush=True)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"FAIL {tag}: {type(e).__name__}: {str(e)[:400]}", flush=True)
print(f"{cases} cases, {fails} failures", flush=True)
