"""Engine: one libbgmf device context (partition + factors + step scratch).

This is the host-side owner of everything that lives in HBM for one GPU:

* the partitioned ratings, SoA ``int32 lrow | int32 lcol | fp32 value``
  (12 B/rating), blocks contiguous in row-major block order, entries of a
  block row-major (the reference's BlockedDataset order);
* U (n x kp) and V (m x kp) fp32, rows padded to kp = ceil(k/4)*4 so every
  row is a whole number of 16-byte vectors (exact mode: fp64, kp = k);
* the per-block SSE array and the divergence word of the current step.

Numbers only ever come back through :meth:`run_step` (P^2 doubles) and the
explicit download calls.
"""

from __future__ import annotations

import ctypes
import os
import sys
import time
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class EngineOptions:
    """B200 knobs.  None of them changes the reference's semantics.

    exact      fp64 sequential-per-block kernels, bit-identical to the
               reference (slow; parity/verification mode).  Default: False,
               or True when $BGMF_EXACT=1 (runs a reference test suite
               unchanged in exact mode, ref_suite/run.py).
    min_chunk  minimum ratings per worker group (bounds concurrency on tiny
               blocks, which keeps the lossless-Hogwild drift far below 1e-3).
    device     CUDA ordinal; default $BGMF_DEVICE, else $LOCAL_RANK, else 0.
    timing     record CUDA events around every kernel launch.
    fused      True: one cooperative launch per outer step (grid barriers
               between strata); False: one launch per stratum sweep / SSE
               pass; None (default): the library's choice (per-stratum
               launches -- faster at every config measured on B200).
    bulk_red   V-row deltas leave through the TMA engine as bulk reduce-adds
               from a shared-memory ring instead of per-lane
               red.global.add.v4.f32.  Off by default: both are bound by the
               SM->L2 request interface on B200 and the per-lane form measured
               ~3% faster (profiles/r01_*).
    sse_wide   post-sweep SSE with 4 ratings' rows in flight per group
               (measured slower than the pipelined walk on C4; off).
    sse_async  post-sweep SSE with the V rows of the next 4 ratings in flight
               per group through a per-lane cp.async shared-memory ring
               (None/True: on; False: the register-pipelined walk).
    l2_wave_bytes
               V-block bytes swept at once: larger strata run as sequential
               waves of blocks whose V fits in L2 (None: library default,
               48 MiB; 0: whole strata).
    ordered    None (default): strata whose blocks' V fits the GPU's shared
               memory run the order-faithful slab sweep (ordered.cu: every U
               and V row updated in the reference's stored order, fp32,
               deterministic); True: the same, stated explicitly; False:
               always the chunked lossless-Hogwild sweep.
    device_rating_budget
               bytes of HBM the ratings may use (None: all resident).  When
               the partition is larger, it moves to pinned host memory and
               every step streams it through ``stream_slots`` device slots
               (out-of-core mode, 12 B per rating per slot entry).
    """

    exact: bool = field(default_factory=lambda: os.environ.get("BGMF_EXACT") == "1")
    min_chunk: int = 256
    device: int | None = None
    timing: bool = False
    warps_per_sm: int = 0
    fused: bool | None = None
    device_rating_budget: int | None = None
    bulk_red: bool = False
    sse_wide: bool = False
    stream_slots: int = 3
    sse_async: bool | None = None
    l2_wave_bytes: int | None = None
    ordered: bool | None = None


def release_host_cache() -> None:
    """Unregister the pinned host buffers cached by closed out-of-core contexts
    (bgmf_release_host_cache)."""
    N.check(N.load().bgmf_release_host_cache(), None)


def default_device() -> int:
    for var in ("BGMF_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v:
            return int(v)
    return 0


class Engine:
    def __init__(self, options: EngineOptions | None = None, *, stream: int | None = None):
        self.options = options or EngineOptions()
        self._L = N.load()
        dev = self.options.device if self.options.device is not None else default_device()
        h = ctypes.c_void_p()
        N.check(self._L.bgmf_create(dev, ctypes.c_void_p(stream or 0), ctypes.byref(h)))
        self._h = h
        self.device = dev
        self._opt("exact", 1.0 if self.options.exact else 0.0)
        self._opt("min_chunk", float(self.options.min_chunk))
        self._opt("timing", 1.0 if self.options.timing else 0.0)
        self._opt("warps_per_sm", float(self.options.warps_per_sm))
        self._opt("bulk_red", 1.0 if self.options.bulk_red else 0.0)
        self._opt("sse_wide", 1.0 if self.options.sse_wide else 0.0)
        self._opt("sse_async", 0.0 if self.options.sse_async is False else 1.0)
        if self.options.ordered is not None:
            self._opt("ordered", 1.0 if self.options.ordered else 0.0)
        if self.options.l2_wave_bytes is not None:
            self._opt("l2_wave_bytes", float(self.options.l2_wave_bytes))
        f = self.options.fused
        self._opt("fused", -1.0 if f is None else (1.0 if f else 0.0))
        # experiments only: raw bgmf_set_option knobs, "key=value,key=value"
        for kv in filter(None, os.environ.get("BGMF_ENGINE_OPTS", "").split(",")):
            key, val = kv.split("=")
            self._opt(key.strip(), float(val))
        self.n = self.m = self.nnz = 0
        self.I = self.J = 0
        self.k = 0
        self.offsets: np.ndarray | None = None

    # ------------------------------------------------------------ plumbing
    def _opt(self, key: str, value: float):
        N.check(self._L.bgmf_set_option(self._h, key.encode(), value), self._h)

    def _check(self, rc: int, **kw):
        N.check(rc, self._h, **kw)

    def close(self):
        pre = getattr(self, "_prefault", None)
        if pre is not None:  # a prefault thread still writing host pages
            pre[0].join()
            self._prefault = None
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.bgmf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, on: bool):
        self._opt("timing", 1.0 if on else 0.0)

    # ------------------------------------------------------------ partition
    def partition(self, rows, cols, values, n: int, m: int, grid_i: int, grid_j: int,
                  data_error=None, row_range: tuple[int, int] | None = None):
        """Partition on the device.  ``row_range=(lo, hi)`` keeps only the
        entries with lo <= row < hi (a multi-GPU rank's shard)."""
        rows, cols, values = N.i64(rows), N.i64(cols), N.f64(values)
        budget = self.options.device_rating_budget
        if (budget is not None and not self.options.exact
                and 12 * self._kept(rows, row_range) > budget):
            # out-of-core: the partition itself stays under the budget (row
            # blocks in chunks straight into the pinned streaming layout)
            slots = self.options.stream_slots
            _t0 = time.perf_counter()
            self._check(self._L.bgmf_partition_ooc(
                self._h, N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(values, N._f64p),
                len(rows), n, m, grid_i, grid_j, int(budget), int(budget // (12 * slots)),
                slots, *(row_range if row_range is not None else (0, -1))),
                data_error=data_error)
            _t1 = time.perf_counter()
            self.I, self.J, self.n, self.m = grid_i, grid_j, n, m
            off = np.zeros(grid_i * grid_j + 1, np.int64)
            self._check(self._L.bgmf_partition_export(self._h, N.ptr(off, N._i64p), None, None,
                                                      None))
            if os.environ.get("BGMF_PROFILE"):
                print(f"[bgmf]   bgmf_partition_ooc call {1e3 * (_t1 - _t0):9.2f} ms, export "
                      f"{1e3 * (time.perf_counter() - _t1):9.2f} ms", file=sys.stderr)
            self.offsets = off
            self.nnz = int(off[-1])
            self.streaming = True
            return
        if row_range is None:
            self._check(self._L.bgmf_partition(
                self._h, N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(values, N._f64p),
                len(rows), n, m, grid_i, grid_j), data_error=data_error)
        else:
            self._check(self._L.bgmf_partition_rows(
                self._h, N.ptr(rows, N._i64p), N.ptr(cols, N._i64p), N.ptr(values, N._f64p),
                len(rows), n, m, grid_i, grid_j, int(row_range[0]), int(row_range[1])),
                data_error=data_error)
        self.I, self.J, self.n, self.m = grid_i, grid_j, n, m
        off = np.zeros(grid_i * grid_j + 1, np.int64)
        self._check(self._L.bgmf_partition_export(self._h, N.ptr(off, N._i64p), None, None, None))
        self.offsets = off
        self.nnz = int(off[-1])
        self.streaming = False
        if budget is not None and 12 * self.nnz > budget:
            slots = self.options.stream_slots
            self.stream(int(budget // (12 * slots)), slots)

    @staticmethod
    def _kept(rows, row_range) -> int:
        """Ratings a (row-ranged) partition keeps -- decides out-of-core mode."""
        if row_range is None:
            return len(rows)
        lo, hi = row_range
        return int(np.count_nonzero((rows >= lo) & (rows < hi)))

    def stream(self, slot_ratings: int, nslots: int = 3):
        """Out-of-core mode: ratings to pinned host memory, `nslots` device slots."""
        self._check(self._L.bgmf_stream_ratings(self._h, int(slot_ratings), int(nslots)))
        self.streaming = True

    def mem_stats(self, reset: bool = False) -> tuple[int, int]:
        """(device pool bytes in use, high-water mark since the last reset)."""
        out = np.zeros(2, np.int64)
        self._check(self._L.bgmf_mem_stats(self._h, N.ptr(out, N._i64p), int(reset)))
        return int(out[0]), int(out[1])

    def streamed_bytes(self) -> float:
        out = ctypes.c_double()
        self._check(self._L.bgmf_stream_stats(self._h, ctypes.byref(out)))
        return out.value

    def export_partition(self):
        """(offsets, order, local rows, local cols) as int64 host arrays."""
        nnz = self.nnz
        off = np.zeros(self.I * self.J + 1, np.int64)
        order = np.empty(nnz, np.int64)
        lr = np.empty(nnz, np.int32)
        lc = np.empty(nnz, np.int32)
        self._check(self._L.bgmf_partition_export(
            self._h, N.ptr(off, N._i64p), N.ptr(order, N._i64p), N.ptr(lr, N._i32p),
            N.ptr(lc, N._i32p)))
        return off, order, lr.astype(np.int64), lc.astype(np.int64)

    def partition_values(self) -> np.ndarray:
        """The device-resident values in partition order, as fp64."""
        out = np.empty(self.nnz, np.float64)
        self._check(self._L.bgmf_partition_values(self._h, N.ptr(out, N._f64p)))
        return out

    # ------------------------------------------------------------ factors
    def set_factors(self, u: np.ndarray, v: np.ndarray):
        u, v = N.f64(u), N.f64(v)
        self._check(self._L.bgmf_set_factors(self._h, N.ptr(u, N._f64p), N.ptr(v, N._f64p),
                                             u.shape[0], v.shape[0], u.shape[1]))
        self.k = u.shape[1]

    def init_factors(self, n: int, m: int, k: int, seed: int):
        """init_factors(n, m, k, seed) generated on the device: the PCG64
        stream of numpy's default_rng(seed), bit-identical (core.py:179-193)."""
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        mask = (1 << 64) - 1
        self._check(self._L.bgmf_init_factors(self._h, s >> 64, s & mask, inc >> 64, inc & mask,
                                              n, m, k))
        self.k = k

    def bind_factors(self, u_ptr: int, v_ptr: int, n: int, m: int, k: int, kp: int):
        self._check(self._L.bgmf_bind_factors(self._h, ctypes.c_void_p(u_ptr),
                                              ctypes.c_void_p(v_ptr), n, m, k, kp))
        self.k = k

    def prefault_factors(self):
        """Allocate get_factors' output arrays now and fault their pages in on
        a side thread (bgmf_host_prefault releases the GIL) while the device
        works; the next get_factors joins it and fills them."""
        u = np.empty((self.n, self.k), np.float64)
        v = np.empty((self.m, self.k), np.float64)

        def touch():
            for a in (u, v):
                self._L.bgmf_host_prefault(a.ctypes.data, a.nbytes)

        t = threading.Thread(target=touch, name="bgmf-prefault", daemon=True)
        t.start()
        self._prefault = (t, u, v)

    def get_factors(self):
        pre, self._prefault = getattr(self, "_prefault", None), None
        if pre is not None:
            pre[0].join()
        if pre is not None and pre[1].shape == (self.n, self.k) and pre[2].shape == (self.m, self.k):
            u, v = pre[1], pre[2]
        else:
            u = np.empty((self.n, self.k), np.float64)
            v = np.empty((self.m, self.k), np.float64)
        self._check(self._L.bgmf_get_factors(self._h, N.ptr(u, N._f64p), N.ptr(v, N._f64p)))
        return u, v

    # ------------------------------------------------------------ steps
    def plan_arrays(self, batches):
        """Plan batches of (bi, bj) -> (flat block ids, batch offsets)."""
        J = self.J
        ids = np.array([bi * J + bj for b in batches for bi, bj in b], np.int32)
        off = np.zeros(len(batches) + 1, np.int32)
        off[1:] = np.cumsum([len(b) for b in batches])
        return ids, off

    def run_step(self, ids: np.ndarray, off: np.ndarray, iters: int, alpha: float, beta: float):
        """Returns (sse[I*J], bad) where bad = (plan_pos, entry, iteration) or None."""
        sse = np.zeros(self.I * self.J, np.float64)
        bad = np.zeros(3, np.int64)
        self._check(self._L.bgmf_run_step(self._h, N.ptr(ids, N._i32p), N.ptr(off, N._i32p),
                                          len(off) - 1, int(iters), float(alpha), float(beta),
                                          N.ptr(sse, N._f64p), N.ptr(bad, N._i64p)))
        return sse, (None if bad[0] < 0 else tuple(int(x) for x in bad))

    def run_step_converge(self, ids, off, tol: float, cap: int, alpha: float, beta: float):
        nb = self.I * self.J
        sse = np.zeros(nb, np.float64)
        iters = np.zeros(nb, np.int64)
        capped = np.zeros(nb, np.int32)
        bad = np.zeros(3, np.int64)
        self._check(self._L.bgmf_run_step_converge(
            self._h, N.ptr(ids, N._i32p), N.ptr(off, N._i32p), len(off) - 1, float(tol),
            int(cap), float(alpha), float(beta), N.ptr(sse, N._f64p), N.ptr(iters, N._i64p),
            N.ptr(capped, N._i32p), N.ptr(bad, N._i64p)))
        return sse, iters, capped, (None if bad[0] < 0 else tuple(int(x) for x in bad))

    def run_steps(self, steps, alpha: float, beta: float):
        """Several outer steps in one call (fast mode): ``steps`` is a list of
        (ids, off, iters) as for run_step.  Returns (sse[nsteps, I*J],
        bad = (step, block id, entry, iteration) or None, device ms per step)."""
        n = len(steps)
        plans = np.concatenate([np.asarray(i, np.int32) for i, _, _ in steps]) if n else \
            np.zeros(1, np.int32)
        offs = np.concatenate([np.asarray(o, np.int32) for _, o, _ in steps]) if n else \
            np.zeros(1, np.int32)
        nbatch = np.array([len(o) - 1 for _, o, _ in steps] or [0], np.int32)
        iters = np.array([int(g) for _, _, g in steps] or [1], np.int32)
        sse = np.zeros((max(n, 1), self.I * self.J), np.float64)
        bad = np.zeros(4, np.int64)
        ms = np.zeros(max(n, 1), np.float32)
        self._check(self._L.bgmf_run_steps(
            self._h, n, N.ptr(plans, N._i32p), N.ptr(offs, N._i32p), N.ptr(nbatch, N._i32p),
            N.ptr(iters, N._i32p), float(alpha), float(beta), N.ptr(sse, N._f64p),
            N.ptr(bad, N._i64p), ms.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return sse[:n], (None if bad[0] < 0 else tuple(int(x) for x in bad)), ms[:n]

    def step_begin(self, max_blocks: int):
        """Asynchronous step (fast mode): reserve ``max_blocks`` block launches."""
        self._check(self._L.bgmf_step_begin(self._h, int(max_blocks)))

    def step_batch(self, ids: np.ndarray, off: np.ndarray, iters: int, alpha: float,
                   beta: float):
        """Enqueue strata (same arrays as run_step); no host synchronisation."""
        self._check(self._L.bgmf_step_batch(self._h, N.ptr(ids, N._i32p), N.ptr(off, N._i32p),
                                            len(off) - 1, int(iters), float(alpha),
                                            float(beta)))

    def step_end(self):
        """(sse[I*J], bad) with bad = (block id, entry, iteration) or None."""
        sse = np.zeros(self.I * self.J, np.float64)
        bad = np.zeros(3, np.int64)
        self._check(self._L.bgmf_step_end(self._h, N.ptr(sse, N._f64p), N.ptr(bad, N._i64p)))
        return sse, (None if bad[0] < 0 else tuple(int(x) for x in bad))

    def step_end_async(self, d_sse: int, d_bad: int):
        """End the step without a host sync: per-block SSEs (fp64 [I*J]) and
        the raw divergence word to the device addresses given."""
        self._check(self._L.bgmf_step_end_async(self._h, ctypes.c_void_p(d_sse),
                                                ctypes.c_void_p(d_bad)))

    # ------------------------------------------------------------ peer transport
    def peer_alloc(self, nbytes: int) -> int:
        """Zeroed IPC-exportable device memory owned by this context."""
        p = ctypes.c_void_p()
        self._check(self._L.bgmf_peer_alloc(self._h, int(nbytes), ctypes.byref(p)))
        return int(p.value)

    def peer_handle(self, base: int) -> bytes:
        buf = ctypes.create_string_buffer(64)
        self._check(self._L.bgmf_peer_handle(self._h, ctypes.c_void_p(base), buf))
        return buf.raw

    def peer_open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        self._check(self._L.bgmf_peer_open(self._h, handle, ctypes.byref(p)))
        return int(p.value)

    def peer_push(self, dst: int, src: int, nbytes: int, peer_flag: int, value: int):
        self._check(self._L.bgmf_peer_push(self._h, ctypes.c_void_p(dst), ctypes.c_void_p(src),
                                           int(nbytes), ctypes.c_void_p(peer_flag),
                                           value & 0xFFFFFFFF))

    def peer_wait(self, flag: int, value: int):
        self._check(self._L.bgmf_peer_wait(self._h, ctypes.c_void_p(flag), value & 0xFFFFFFFF))

    def peer_config(self, abort_word: int, timeout_s: float):
        self._check(self._L.bgmf_peer_config(self._h, ctypes.c_void_p(abort_word),
                                             float(timeout_s)))

    def peer_abort(self, peer_abort_word: int):
        self._check(self._L.bgmf_peer_abort(self._h, ctypes.c_void_p(peer_abort_word)))

    def peer_error(self) -> int:
        """0, 1 (a peer wait timed out) or 2 (a peer aborted the ring)."""
        out = ctypes.c_int(0)
        self._check(self._L.bgmf_peer_error(self._h, ctypes.byref(out)))
        return int(out.value)

    def run_sync_parallel_step(self, edges: np.ndarray, alpha: float, beta: float):
        """CPMF step on a 1x1 partition; returns (per-shard SSE, bad) where
        bad = (shard, entry, iteration) or None."""
        edges = np.ascontiguousarray(edges, np.int64)
        ns = len(edges) - 1
        sse = np.zeros(ns, np.float64)
        bad = np.zeros(3, np.int64)
        self._check(self._L.bgmf_run_sync_parallel_step(
            self._h, N.ptr(edges, N._i64p), ns, float(alpha), float(beta),
            N.ptr(sse, N._f64p), N.ptr(bad, N._i64p)))
        return sse, (None if bad[0] < 0 else tuple(int(x) for x in bad))

    def train_sse(self) -> float:
        out = ctypes.c_double()
        self._check(self._L.bgmf_train_sse(self._h, ctypes.byref(out)))
        return out.value

    # ------------------------------------------------------------ holdout
    def holdout_set(self, rows, cols, values, cold: np.ndarray, fallback: float):
        rows, cols, values = N.i64(rows), N.i64(cols), N.f64(values)
        cold = np.ascontiguousarray(cold, np.uint8)
        self._check(self._L.bgmf_holdout_set(self._h, N.ptr(rows, N._i64p), N.ptr(cols, N._i64p),
                                             N.ptr(values, N._f64p), N.ptr(cold, N._u8p),
                                             len(rows), float(fallback)))
        self._hcount = len(rows)

    def holdout_sse(self) -> float:
        out = ctypes.c_double()
        self._check(self._L.bgmf_holdout_sse(self._h, ctypes.byref(out)))
        return out.value

    # ------------------------------------------------------------ timing
    def kernel_stats(self, reset: bool = False) -> dict:
        out = np.zeros(5, np.float64)
        self._check(self._L.bgmf_kernel_stats(self._h, N.ptr(out, N._f64p), 1 if reset else 0))
        return dict(sgd_ms=out[0], sse_ms=out[1], sgd_launches=int(out[2]),
                    sse_launches=int(out[3]), sgd_alg_bytes=out[4])
