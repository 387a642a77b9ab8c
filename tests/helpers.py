"""Test helpers: dataset reconstruction for golden traces, hashing."""

import hashlib

import numpy as np

import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_inputs(name: str):
    """(train dataset, test dataset or None) of a golden trace case."""
    if "holdout" in name and name.startswith(("cpmf", "cmf")):
        d = bm.gen_synthetic(bm.SyntheticSpec(64, 64, 1, 30, seed=0))
        return bm.split(d, 0.2, seed=1)
    if name.startswith(("c1", "cmf_c1", "cpmf_c1")):
        d = workloads.ml100k_dataset()
        if name == "c1_split":
            return bm.split(d, 0.2, seed=0)
        return d, None
    d = bm.gen_synthetic(bm.SyntheticSpec(64, 64, 1, 30, seed=0))
    if name == "dense64_holdout":
        return bm.split(d, 0.2, seed=1)
    return d, None


def config_of(meta) -> bm.TrainConfig:
    c = meta["cfg"]
    return bm.TrainConfig(k=c["k"], alpha=c["alpha"], beta=c["beta"], delta=c["delta"],
                          outer_steps=c["outer_steps"],
                          inner_schedule=bm.parse_schedule(c["schedule"]),
                          grid_i=c["grid_i"], grid_j=c["grid_j"], seed=c["seed"])


def baseline_config(meta) -> bm.TrainConfig:
    c = meta["cfg"]
    return bm.TrainConfig(k=c["k"], alpha=c["alpha"], beta=c["beta"], delta=c["delta"],
                          outer_steps=c["outer_steps"], seed=c["seed"], workers=c["workers"],
                          inner_schedule=bm.parse_schedule(c["schedule"]),
                          grid_i=c["grid_i"], grid_j=c["grid_j"])
