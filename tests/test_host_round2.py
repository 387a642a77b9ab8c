"""Host-side pieces added in round 2 (no GPU): the skewed workload generator,
the exact-mode environment default, and the reference-suite alias."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2304_13724_b200 as bm
from paper_2304_13724_b200 import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_zipf_cells_distinct_deterministic_heavy_tailed():
    a = workloads.zipf_cells(20_000, 3_000, 200_000, seed=3, device="cpu")
    b = workloads.zipf_cells(20_000, 3_000, 200_000, seed=3, device="cpu")
    assert len(a) == 200_000 and len(np.unique(a)) == 200_000
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() < 20_000 * 3_000
    items = np.bincount(a % 3_000, minlength=3_000)
    users = np.bincount(a // 3_000, minlength=20_000)
    assert items.max() > 20 * np.median(items)  # hot items
    assert users.max() > 10 * max(np.median(users), 1)  # heavy users


def test_exact_default_from_environment(monkeypatch):
    monkeypatch.delenv("BGMF_EXACT", raising=False)
    assert bm.EngineOptions().exact is False
    monkeypatch.setenv("BGMF_EXACT", "1")
    assert bm.EngineOptions().exact is True
    assert bm.EngineOptions(exact=False).exact is False


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/tests"),
                    reason="the reference's tests are only present in the build container")
def test_reference_host_suites_through_alias():
    """ref_suite/run.py runs the reference's own tests with `blockmf` aliased to
    this package; the host-only suites (value types, the stratum schedule;
    FactorModel.predict runs on the GPU, so it is left out) pass here."""
    subprocess.run([sys.executable, os.path.join(ROOT, "ref_suite", "run.py"), "sync"],
                   check=True, capture_output=True)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "ref_suite", "run.py"), "fast",
                        "test_scheduler.py", "test_core.py", "-k", "not predict"],
                       capture_output=True, text=True, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:]
    assert " passed" in p.stdout
