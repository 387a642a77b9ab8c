"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and call the CUDA path
through the C ABI; everything else runs on CPU (oracle vs golden vectors,
host logic, ABI symbol checks)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_13724_b200 as bm  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

try:
    from hypothesis import settings

    settings.register_profile("suite", deadline=None, max_examples=50)
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libbgmf.so")
    config.addinivalue_line("markers", "slow: large (C3/C4-sized) parity or property test")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kernel_cases():
    return np.load(os.path.join(GOLDEN, "kernel_cases.npz"))


@pytest.fixture(scope="session")
def partition_cases():
    return np.load(os.path.join(GOLDEN, "partition_cases.npz"))


@pytest.fixture(scope="session")
def baseline_cases():
    return np.load(os.path.join(GOLDEN, "baseline_cases.npz"))


@pytest.fixture(scope="session")
def train_cases():
    return np.load(os.path.join(GOLDEN, "train_cases.npz"))


def dense(n):
    return bm.gen_synthetic(bm.SyntheticSpec(n, n, 1, 30, seed=0))


@pytest.fixture(scope="session")
def dense32():
    return dense(32)


@pytest.fixture(scope="session")
def dense64():
    return dense(64)


@pytest.fixture(scope="session")
def dense256():
    return dense(256)


@pytest.fixture(scope="session")
def standin():
    from paper_2304_13724_b200 import workloads

    return workloads.ml100k_dataset()
