"""The C ABI library loads and exports every symbol include/bgmf.h declares
(no compute calls: this runs on the CPU-only build container too)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2304_13724_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bgmf.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bgmf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("bgmf_partition", "bgmf_run_step", "bgmf_sgd_sweeps", "bgmf_sgd_converge",
              "bgmf_block_sse", "bgmf_sse", "bgmf_predict", "bgmf_holdout_sse"):
        assert s in syms


def test_signatures_cover_header():
    assert sorted(N.SIGNATURES) == declared_symbols()


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(N.LIB_PATH):
        pytest.fail("libbgmf.so is not built (run __graft_entry__.build())")
    L = N.load()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.bgmf_version() == 100


def test_dynamic_symbol_table():
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (bgmf_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_targets_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_without_context_are_reported():
    L = N.load()
    rc = L.bgmf_set_option(None, b"exact", 1.0)
    assert rc == N.ERR_ARG
    assert L.bgmf_last_error(None)
    ctx = ctypes.c_void_p()
    assert L.bgmf_create(-1, None, ctypes.byref(ctx)) != 0


def test_host_prefault_zero_fills_without_a_gpu():
    """bgmf_host_prefault is host-only (no CUDA call): it faults in and
    zero-fills one byte per 4 KiB page of a caller buffer."""
    import numpy as np

    lib = N.load()
    a = np.full(3 * 1024 * 1024 + 123, 7, np.uint8)  # spans 2 MiB pages, ragged tail
    assert lib.bgmf_host_prefault(a.ctypes.data, a.nbytes) == 0
    assert (a[::4096] == 0).all()
    assert lib.bgmf_host_prefault(None, 0) == 0
