"""ctypes binding of ``libbgmf.so`` (C ABI declared in ``include/bgmf.h``).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every numeric entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbgmf.so")

OK, ERR_CUDA, ERR_ARG, ERR_STATE, ERR_DATA, ERR_NOMEM = 0, -1, -2, -3, -4, -5


class NativeUnavailable(RuntimeError):
    """libbgmf.so could not be loaded (not built, or no CUDA runtime)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libbgmf.so."""


_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p
_ctx = ctypes.c_void_p
_i, _l, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_double

# name -> (restype, argtypes); every symbol include/bgmf.h declares
SIGNATURES = {
    "bgmf_version": (_i, []),
    "bgmf_probe_l2": (_i, [_i, _l, _l, _i, _i, _f64p]),
    "bgmf_probe_dsmem": (_i, [_i, _l, _l, _i, _i, _i, _f64p]),
    "bgmf_create": (_i, [_i, _vp, ctypes.POINTER(_ctx)]),
    "bgmf_destroy": (None, [_ctx]),
    "bgmf_last_error": (ctypes.c_char_p, [_ctx]),
    "bgmf_set_option": (_i, [_ctx, ctypes.c_char_p, _d]),
    "bgmf_partition": (_i, [_ctx, _i64p, _i64p, _f64p, _l, _l, _l, _i, _i]),
    "bgmf_partition_export": (_i, [_ctx, _i64p, _i64p, _i32p, _i32p]),
    "bgmf_partition_values": (_i, [_ctx, _f64p]),
    "bgmf_release_host_cache": (_i, []),
    "bgmf_synth_partition": (_i, [_ctx, _l, _l, _l, ctypes.c_uint64, _i, _i]),
    "bgmf_synth": (_i, [_l, _l, _l, _l, ctypes.c_uint64, _i64p, _i64p, _f64p]),
    "bgmf_set_factors": (_i, [_ctx, _f64p, _f64p, _l, _l, _i]),
    "bgmf_get_factors": (_i, [_ctx, _f64p, _f64p]),
    "bgmf_host_prefault": (_i, [ctypes.c_void_p, ctypes.c_int64]),
    "bgmf_init_factors": (_i, [_ctx, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_uint64, _l, _l, _i]),
    "bgmf_bind_factors": (_i, [_ctx, _vp, _vp, _l, _l, _i, _i]),
    "bgmf_run_step": (_i, [_ctx, _i32p, _i32p, _i, _i, _d, _d, _f64p, _i64p]),
    "bgmf_partition_rows": (_i, [_ctx, _i64p, _i64p, _f64p, _l, _l, _l, _i, _i, _l, _l]),
    "bgmf_run_steps": (_i, [_ctx, _i, _i32p, _i32p, _i32p, _i32p, _d, _d, _f64p, _i64p,
                            ctypes.POINTER(ctypes.c_float)]),
    "bgmf_step_begin": (_i, [_ctx, _i]),
    "bgmf_step_batch": (_i, [_ctx, _i32p, _i32p, _i, _i, _d, _d]),
    "bgmf_step_end": (_i, [_ctx, _f64p, _i64p]),
    "bgmf_step_end_async": (_i, [_ctx, ctypes.c_void_p, ctypes.c_void_p]),
    "bgmf_peer_alloc": (_i, [_ctx, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "bgmf_peer_handle": (_i, [_ctx, ctypes.c_void_p, ctypes.c_char_p]),
    "bgmf_peer_open": (_i, [_ctx, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bgmf_peer_push": (_i, [_ctx, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_void_p, ctypes.c_uint32]),
    "bgmf_peer_wait": (_i, [_ctx, ctypes.c_void_p, ctypes.c_uint32]),
    "bgmf_peer_config": (_i, [_ctx, ctypes.c_void_p, ctypes.c_double]),
    "bgmf_peer_abort": (_i, [_ctx, ctypes.c_void_p]),
    "bgmf_peer_error": (_i, [_ctx, ctypes.POINTER(ctypes.c_int)]),
    "bgmf_run_sync_parallel_step": (_i, [_ctx, _i64p, _i, _d, _d, _f64p, _i64p]),
    "bgmf_run_step_converge": (_i, [_ctx, _i32p, _i32p, _i, _d, _l, _d, _d, _f64p, _i64p,
                                    _i32p, _i64p]),
    "bgmf_train_sse": (_i, [_ctx, _f64p]),
    "bgmf_holdout_set": (_i, [_ctx, _i64p, _i64p, _f64p, _u8p, _l, _d]),
    "bgmf_holdout_sse": (_i, [_ctx, _f64p]),
    "bgmf_kernel_stats": (_i, [_ctx, _f64p, _i]),
    "bgmf_stream_ratings": (_i, [_ctx, _l, _i]),
    "bgmf_mem_stats": (_i, [_ctx, _i64p, _i]),
    "bgmf_partition_ooc": (_i, [_ctx, _i64p, _i64p, _f64p, _l, _l, _l, _i, _i, _l, _l, _i, _l,
                                _l]),
    "bgmf_stream_stats": (_i, [_ctx, _f64p]),
    "bgmf_sgd_sweeps": (_i, [_i64p, _i64p, _f64p, _l, _f64p, _l, _f64p, _l, _i, _d, _d, _i,
                             _f64p, _f64p, _i64p, _i64p]),
    "bgmf_gradient_steps": (_i, [_i64p, _i64p, _f64p, _l, _f64p, _l, _f64p, _l, _i, _d, _d, _i,
                                 _f64p, _f64p, _i64p, _i64p]),
    "bgmf_block_gradients": (_i, [_i64p, _i64p, _f64p, _l, _f64p, _l, _f64p, _l, _i, _d, _f64p,
                                  _f64p, _f64p, _f64p]),
    "bgmf_sgd_converge": (_i, [_i64p, _i64p, _f64p, _l, _f64p, _l, _f64p, _l, _i, _d, _d, _d,
                               _l, _f64p, _f64p, _i64p, _i32p, _i64p, _i64p]),
    "bgmf_block_sse": (_i, [_i64p, _i64p, _f64p, _l, _f64p, _l, _f64p, _l, _i, _f64p]),
    "bgmf_predict": (_i, [_f64p, _l, _f64p, _l, _i, _i64p, _i64p, _l, _f64p]),
    "bgmf_sse": (_i, [_f64p, _l, _f64p, _l, _i, _i64p, _i64p, _f64p, _u8p, _d, _l, _f64p]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libbgmf.so and declare its signatures (no CUDA call is made)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeUnavailable(
                    f"{path} is not built; run `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (nvcc, sm_100a)")
            try:
                L = ctypes.CDLL(path)
            except OSError as exc:  # missing libcudart etc.
                raise NativeUnavailable(f"cannot load {path}: {exc}") from None
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def error_message(ctx) -> str:
    msg = load().bgmf_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None, *, data_error=None):
    """Map a BGMF_ERR_* code to the reference's exception types."""
    if rc == OK:
        return
    msg = error_message(ctx) or f"libbgmf error {rc}"
    if rc == ERR_DATA:
        if data_error is None:
            from .core import DataError as data_error  # noqa: N813
        raise data_error(msg)
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_STATE:
        raise RuntimeError(msg)
    if rc == ERR_NOMEM:
        raise MemoryError(msg)
    if "no CUDA-capable device" in msg or "cudaErrorNoDevice" in msg or \
            "cudaErrorInsufficientDriver" in msg:
        raise NativeUnavailable(msg)
    raise CudaError(msg)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
