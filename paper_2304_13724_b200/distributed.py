"""Multi-GPU BGMF: one process per GPU, U resident, V blocks rotating.

SURVEY §8(e).  A stratum's blocks own pairwise-disjoint U and V slices, so the
result does not depend on which GPU computes which block.  Rank g owns the
contiguous U row-blocks ``[g*R, (g+1)*R)`` (R = ceil(I / G)) and all rating
blocks of those rows (≈ nnz/G ratings and n/G U rows stay in its HBM).  For the
square rotating plan, batch t of step s pairs row-block r with column
(r - s - t) mod P, so after every batch each V block moves one row down: G
blocks per batch cross to rank g+1, and at a step boundary every block moves
two rows.  :class:`RingSchedule` derives those transfers generically from any
plan (`plan_step` of any I x J grid), so wide grids work too.

Transfers are NCCL point-to-point (``torch.distributed`` batch_isend_irecv of V
slices that the engine uses in place via ``bgmf_bind_factors``) ordered on the
engine's CUDA stream.  Per-block SSEs are summed across ranks (all-reduce of
P^2 doubles) and merged in plan order on every rank, exactly like the
single-GPU trainer.  The same schedule code drives the CPU/gloo tests, where
the per-block compute is the oracle (tests only).
"""

from __future__ import annotations

import math
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

from .scheduler import plan_step


@dataclass(frozen=True)
class Transfer:
    col: int   # V column-block
    src: int   # rank holding its latest version
    dst: int   # rank that needs it for the next batch


class RingSchedule:
    """Row-block ownership and the V-block moves implied by the plans."""

    def __init__(self, grid_i: int, grid_j: int, world: int):
        if world < 1:
            raise ValueError("world must be >= 1")
        self.I, self.J, self.G = grid_i, grid_j, world
        self.R = math.ceil(grid_i / world)
        # holder[j]: rank with the latest V_j; None = every rank (initial replicas)
        self.holder: list[int | None] = [None] * grid_j

    def owner(self, bi: int) -> int:
        return min(bi // self.R, self.G - 1)

    def rows_of(self, rank: int) -> range:
        lo = min(rank * self.R, self.I)
        hi = self.I if rank == self.G - 1 else min((rank + 1) * self.R, self.I)
        return range(lo, hi)

    def batches(self, step0: int):
        return [list(b) for b in plan_step(self.I, self.J, step0)]

    def transfers_for(self, batch) -> list[Transfer]:
        """Moves needed before ``batch`` runs; updates the holders."""
        moves = []
        for bi, bj in batch:
            dst = self.owner(bi)
            src = self.holder[bj]
            if src is not None and src != dst:
                moves.append(Transfer(bj, src, dst))
            self.holder[bj] = dst
        return moves

    def local_blocks(self, batch, rank: int):
        return [(bi, bj) for bi, bj in batch if self.owner(bi) == rank]


def _staged(dist, t) -> bool:
    """CUDA tensor on a non-NCCL process group (gloo: several ranks sharing one
    GPU in tests): collectives go through host copies."""
    return getattr(t, "is_cuda", False) and dist.get_backend() != "nccl"


def _all_reduce(dist, t, op=None) -> None:
    op = dist.ReduceOp.SUM if op is None else op
    if _staged(dist, t):
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)


def _broadcast(dist, t, src: int) -> None:
    if _staged(dist, t):
        h = t.cpu()
        dist.broadcast(h, src=src)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src)


def exchange(moves, rank: int, v_slice, dist) -> None:
    """Run one batch's V moves: isend what this rank holds, irecv what it needs.
    On NCCL the moves are ordered on the current stream (no host wait); on gloo
    with CUDA tensors they are staged through host buffers."""
    ops, back = [], []
    for mv in moves:
        if mv.src == rank:
            t = v_slice(mv.col)
            ops.append(dist.P2POp(dist.isend, t.cpu() if _staged(dist, t) else t, mv.dst))
        elif mv.dst == rank:
            t = v_slice(mv.col)
            if _staged(dist, t):
                h = t.new_empty(t.shape, device="cpu")
                back.append((t, h))
                t = h
            ops.append(dist.P2POp(dist.irecv, t, mv.src))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for t, h in back:
        t.copy_(h)


def sync_all_v(sched: RingSchedule, rank: int, v_slice, dist) -> None:
    """Give every rank the latest version of every V block (broadcast from holders)."""
    for j in range(sched.J):
        src = sched.holder[j]
        if src is not None:
            _broadcast(dist, v_slice(j), src)


def shard_rows(rows: np.ndarray, row_bounds: np.ndarray, sched: RingSchedule, rank: int):
    """Mask of the ratings whose row-block this rank owns."""
    r = sched.rows_of(rank)
    lo, hi = row_bounds[r.start], row_bounds[r.stop]
    return (rows >= lo) & (rows < hi)


def run_epoch(sched: RingSchedule, shard, rank: int, dist, step0: int, g: int,
              alpha: float, beta: float, nb: int, J: int):
    """One outer step on this rank: before each batch move the V blocks it
    needs, then run the batch's blocks whose rows this rank owns.  Returns
    (local per-block SSE [nb], plan order of block ids, first local divergence
    as (block, entry, iter) or None).  ``shard`` provides ``v_slice(j)`` and
    ``run_batch(blocks, g, alpha, beta)``, which either returns
    ``(sse[nb], bad, ids)`` (synchronous shards) or None when the shard is
    asynchronous: then ``begin_epoch(max_blocks)`` / ``end_epoch() -> (sse[nb],
    bad)`` bracket the step and nothing waits on the host between batches
    (the GPU shard: V moves and strata are ordered on one CUDA stream)."""
    sse_all = np.zeros(nb, np.float64)
    order: list[int] = []
    bad_any = None
    begin = getattr(shard, "begin_epoch", None)
    if begin is not None:
        begin(nb)
    for batch in sched.batches(step0):
        _move_v(sched.transfers_for(batch), rank, shard, dist)
        order.extend(bi * J + bj for bi, bj in batch)
        mine = sched.local_blocks(batch, rank)
        if mine:
            res = shard.run_batch(mine, g, alpha, beta)
            if res is not None:
                sse, bad, ids = res
                sse_all[ids] = sse[ids]
                if bad is not None and bad_any is None:
                    bad_any = (int(ids[bad[0]]), bad[1], bad[2])
    end = getattr(shard, "end_epoch", None)
    if end is not None:
        sse_all, bad_any = end()
    return sse_all, order, bad_any


def _run_epochs_batched(sched: RingSchedule, shard, rank: int, dist, cfg, nb: int,
                        device: int, timing: bool):
    """Every outer step of a run with a fixed inner schedule, no early
    stopping and no holdout set, without a host round trip between steps:
    each step's per-block SSEs and divergence word stay in HBM
    (bgmf_step_end_async) and are all-reduced there (NCCL, ordered on the
    engine stream), so the host keeps enqueueing V moves and strata while the
    GPUs work; every step's results are read once at the end.  Returns, per
    step, (global sse[nb], plan order, local divergence as (block, entry,
    iter) or None, any rank diverged, inner iterations, seconds)."""
    import torch

    from .trainer import resolve_inner_iters

    S, J = cfg.outer_steps, cfg.grid_j
    dev = f"cuda:{device}"
    sse = torch.zeros((S, nb), dtype=torch.float64, device=dev)
    bad = torch.full((S,), -1, dtype=torch.int64, device=dev)  # all ones = clean
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(S + 1)] if timing else None
    if ev:
        ev[0].record(shard.stream)
    orders, subs, gs = [], [], []
    for k in range(S):
        g = resolve_inner_iters(cfg.inner_schedule, k + 1, 1.0)
        order: list[int] = []
        shard.begin_epoch(nb)
        for batch in sched.batches(k):
            _move_v(sched.transfers_for(batch), rank, shard, dist)
            order.extend(bi * J + bj for bi, bj in batch)
            mine = sched.local_blocks(batch, rank)
            if mine:
                shard.run_batch(mine, g, cfg.alpha, cfg.beta)
        subs.append(shard.end_epoch_async(sse[k], bad[k]))
        _all_reduce(dist, sse[k])
        orders.append(order)
        gs.append(g)
        if ev:
            ev[k + 1].record(shard.stream)
    flag = (bad != -1).to(torch.int64)
    _all_reduce(dist, flag, dist.ReduceOp.MAX)
    sse_h, bad_h, flag_h = sse.cpu().numpy(), bad.cpu().numpy(), flag.cpu().numpy()
    out = []
    for k in range(S):
        local = None
        if int(bad_h[k]) != -1:
            w = int(bad_h[k]) & 0xFFFFFFFFFFFFFFFF
            pos, it, entry = w >> 48, (w >> 32) & 0xFFFF, w & 0xFFFFFFFF
            local = (subs[k][pos] if pos < len(subs[k]) else -1, entry, it)
        secs = ev[k].elapsed_time(ev[k + 1]) / 1e3 if ev else 0.0
        out.append((sse_h[k], orders[k], local, bool(flag_h[k]), gs[k], secs))
    return out


def _run_epoch_converge(sched: RingSchedule, shard, rank: int, dist, step0: int, tol: float,
                        alpha: float, beta: float, nb: int, J: int):
    """run_epoch for ConvergeEachBlock: each stratum's local blocks sweep until
    their RMSE improves by < tol (cap CONVERGE_CAP, _kernels.py:62-100);
    synchronous per batch.  Also returns every local block's sweep count and
    the number of capped blocks."""
    from .kernel import CONVERGE_CAP

    sse_all = np.zeros(nb, np.float64)
    order: list[int] = []
    bad_any = None
    iters_used = []
    capped = 0
    for batch in sched.batches(step0):
        _move_v(sched.transfers_for(batch), rank, shard, dist)
        order.extend(bi * J + bj for bi, bj in batch)
        mine = sched.local_blocks(batch, rank)
        if mine:
            ids, off = shard.eng.plan_arrays([mine])
            sse, its, cap, bad = shard.eng.run_step_converge(ids, off, tol, CONVERGE_CAP, alpha,
                                                             beta)
            sse_all[ids] = sse[ids]
            iters_used.extend(int(its[b]) for b in ids)
            capped += int(sum(int(cap[b]) for b in ids))
            if bad is not None and bad_any is None:
                bad_any = (int(ids[bad[0]]), bad[1], bad[2])
    return sse_all, order, bad_any, np.array(iters_used, np.int64), capped


# ---------------------------------------------------------------------------- GPU


class _DeviceArray:
    """A raw device allocation seen by torch (``torch.as_tensor``) through
    ``__cuda_array_interface__``; the memory stays owned by the engine."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


class _PeerLinks:
    """The ring's V moves over peer memory (csrc/peer.cu): every rank maps the
    other ranks' V buffers and flag words once (CUDA IPC handles exchanged with
    all_gather_object); a move src -> dst is a copy into dst's V rows plus a
    release-store of the link's sequence number into dst's flag[src], and dst's
    stream waits for that number before its next sweep."""

    def __init__(self, eng, vptr: int, kp: int, col_bounds, dist):
        self.eng, self.vptr, self.kp, self.cb = eng, vptr, kp, col_bounds
        world, rank = dist.get_world_size(), dist.get_rank()
        self.rank = rank
        # flags[s]: moves s -> me done; flags[world]: the ring's abort word
        self.flags = eng.peer_alloc(4 * (world + 1))
        self.world = world
        eng.peer_config(self.flags + 4 * world,
                        float(os.environ.get("BGMF_PEER_TIMEOUT_S", "120")))
        mine = (eng.peer_handle(vptr), eng.peer_handle(self.flags))
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        self.peer_v, self.peer_flags = {}, {}
        for r in range(world):
            if r != rank:
                self.peer_v[r] = eng.peer_open(allh[r][0])
                self.peer_flags[r] = eng.peer_open(allh[r][1])
        self.sent = [0] * world
        self.got = [0] * world
        dist.barrier()  # every rank's flags are zero and mapped before any move

    def abort(self) -> None:
        """This rank is failing: release every peer's waits on it."""
        for r, f in self.peer_flags.items():
            try:
                self.eng.peer_abort(f + 4 * self.world)
            except Exception:  # noqa: BLE001  best effort on the error path
                pass

    def check(self) -> None:
        """Raise if a wait of this rank gave up (peer dead or aborted)."""
        e = self.eng.peer_error()
        if e:
            raise RuntimeError("ring V move: " + ("a peer rank stopped responding (wait timed "
                               "out)" if e == 1 else "a peer rank aborted the ring"))

    def move(self, moves) -> None:
        """One batch's moves: all pushes first, then the waits (a wait blocks
        the stream; pushing after it could deadlock two ranks)."""
        for mv in moves:
            if mv.src == self.rank:
                self.sent[mv.dst] += 1
                lo, hi = int(self.cb[mv.col]), int(self.cb[mv.col + 1])
                off, nbytes = lo * self.kp * 4, (hi - lo) * self.kp * 4
                self.eng.peer_push(self.peer_v[mv.dst] + off, self.vptr + off, nbytes,
                                   self.peer_flags[mv.dst] + 4 * self.rank, self.sent[mv.dst])
        for mv in moves:
            if mv.dst == self.rank:
                self.got[mv.src] += 1
                self.eng.peer_wait(self.flags + 4 * mv.src, self.got[mv.src])


def _transport(world: int, device: int | None = None, dist=None) -> str:
    """V-move transport of the ring: "peer" (IPC-mapped peer memory,
    csrc/peer.cu) when every rank is on this node and every rank's GPU can
    reach every other's; else "dist" (torch.distributed P2P).
    BGMF_RING_TRANSPORT overrides.  Launchers that do not say how many ranks
    share the node (no LOCAL_WORLD_SIZE: mpirun, custom launchers) get "dist"."""
    if world <= 1:
        return "dist"  # nothing moves
    lws = os.environ.get("LOCAL_WORLD_SIZE")
    single_node = lws is not None and int(lws) == world
    t = os.environ.get("BGMF_RING_TRANSPORT")
    if t is None:
        t = "peer" if single_node and _peers_reachable(world, device, dist) else "dist"
    return "dist" if t in ("dist", "nccl") else t


def _peers_reachable(world: int, device, dist) -> bool:
    """Collective: can every rank's GPU map every other rank's memory (CUDA
    IPC + P2P)?  Ranks sharing one device are fine."""
    if device is None or dist is None:
        return True
    import torch

    devs = [None] * world
    dist.all_gather_object(devs, int(device))
    ok = all(o == device or torch.cuda.can_device_access_peer(device, o) for o in devs)
    ok = _all_ok(ok, device, dist)
    if ok:  # and CUDA IPC itself works here (containers can forbid it)
        ok = _all_ok(_ipc_probe(world, device, dist), device, dist)
    return ok


def _all_ok(ok: bool, device, dist) -> bool:
    import torch

    flag = torch.tensor([1 if ok else 0], dtype=torch.int64,
                        device=f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(int(flag.item()))


def _ipc_probe(world: int, device, dist) -> bool:
    """Collective: export a small peer buffer, map every other rank's.  Any
    failure (on any rank) makes the ring fall back to torch.distributed."""
    from .device import Engine, EngineOptions

    eng = None
    ok, handle = True, None
    try:
        eng = Engine(EngineOptions(device=device))
        handle = eng.peer_handle(eng.peer_alloc(256))
    except Exception:  # noqa: BLE001  probing: any failure means "no peer transport"
        ok = False
    allh = [None] * world
    dist.all_gather_object(allh, handle)
    if ok:
        try:
            for h in allh:
                if h is None:
                    ok = False
                elif h != handle:
                    eng.peer_open(h)
        except Exception:  # noqa: BLE001
            ok = False
    ok = _all_ok(ok, device, dist)  # nobody closes while a peer may still map it
    if eng is not None:
        eng.close()
    return ok


def _move_v(moves, rank: int, shard, dist) -> None:
    """A batch's V moves: over peer memory when the shard has links, else
    through torch.distributed (NCCL P2P, or gloo staged through the host)."""
    peer = getattr(shard, "peer", None)
    if peer is not None:
        peer.move(moves)
    else:
        exchange(moves, rank, shard.v_slice, dist)


class GpuShard:
    """This rank's engine: its ratings and full-size U/V buffers, bound into
    libbgmf with bgmf_bind_factors.  U is a torch tensor; V too for the "dist"
    transport (NCCL moves V slices), or IPC-exportable engine memory seen as a
    torch tensor for the "peer" transport (peers write moved blocks into it)."""

    def __init__(self, d, cfg, sched: RingSchedule, rank: int, device: int, options=None,
                 transport: str = "dist", dist=None):
        import torch

        from .device import Engine, EngineOptions
        from .partition import make_grid

        self.torch = torch
        self.grid = make_grid(d.n, d.m, cfg.grid_i, cfg.grid_j)
        self.stream = torch.cuda.current_stream(device)
        if self.stream.cuda_stream == 0:
            raise RuntimeError("GpuShard needs a non-default current stream (torch.cuda.stream(...)):"
                               " its kernels, the V moves and torch ops must share it")
        opts = options or EngineOptions()
        if opts.exact:
            raise ValueError("the multi-GPU ring runs the fast kernels only; exact (fp64, "
                             "reference-order) training is single-GPU: train_blocked")
        opts = EngineOptions(exact=False, min_chunk=opts.min_chunk, device=device,
                             timing=opts.timing, warps_per_sm=opts.warps_per_sm,
                             device_rating_budget=opts.device_rating_budget,
                             stream_slots=opts.stream_slots, ordered=opts.ordered)
        self.eng = Engine(opts, stream=self.stream.cuda_stream)
        # a rank sweeps a stratum's blocks of its own rows (C4 on 8 GPUs: 2
        # per batch), so the chunked kernel runs more groups per V row than a
        # whole-stratum launch; csrc/ordered.cu use_ordered
        self.eng._opt("ord_col_conc", float(os.environ.get("BGMF_RING_COL_CONC", "6")))
        # this rank's U row-blocks: the upload keeps only their ratings
        # (bgmf_partition_rows), no host-side gather of the dataset
        own = sched.rows_of(rank)
        rb = self.grid.row_bounds
        t0 = time.perf_counter()
        self.eng.partition(d.rows, d.cols, d.values, d.n, d.m, cfg.grid_i, cfg.grid_j,
                           row_range=(int(rb[own.start]), int(rb[own.stop])))
        if os.environ.get("BGMF_PROFILE"):
            print(f"[bgmf]   shard partition call {1e3 * (time.perf_counter() - t0):.2f} ms",
                  file=sys.stderr)
        self.local_nnz = self.eng.nnz
        self.k, self.kp = cfg.k, (cfg.k + 3) // 4 * 4
        self.U = torch.zeros((d.n, self.kp), dtype=torch.float32, device=f"cuda:{device}")
        self.peer = None
        if transport == "peer":  # else "dist": torch.distributed P2P (NCCL, or staged gloo)
            # V in IPC-exportable memory; peers write moved blocks straight into it
            vptr = self.eng.peer_alloc(d.m * self.kp * 4)
            self.V = torch.as_tensor(_DeviceArray(vptr, (d.m, self.kp), "<f4"),
                                     device=f"cuda:{device}")
            self.peer = _PeerLinks(self.eng, vptr, self.kp, self.grid.col_bounds, dist)
        else:
            self.V = torch.zeros((d.m, self.kp), dtype=torch.float32, device=f"cuda:{device}")
        self.eng.bind_factors(self.U.data_ptr(), self.V.data_ptr(), d.n, d.m, cfg.k, self.kp)
        self.counts = np.diff(self.eng.offsets)

    def set_factors(self, u, v):
        self.eng.set_factors(u, v)

    def v_slice(self, j: int):
        cb = self.grid.col_bounds
        return self.V[int(cb[j]):int(cb[j + 1])]

    def u_rows(self, rows: range):
        rb = self.grid.row_bounds
        return self.U[int(rb[rows.start]):int(rb[rows.stop])]

    def begin_epoch(self, max_blocks: int):
        self.eng.step_begin(max_blocks)
        self.submitted: list[tuple[int, int]] = []

    def run_batch(self, blocks, g: int, alpha: float, beta: float):
        """Enqueue this rank's blocks of one stratum (no host sync)."""
        ids, off = self.eng.plan_arrays([blocks])
        self.eng.step_batch(ids, off, g, alpha, beta)
        self.submitted.extend(int(b) for b in ids)
        return None

    def end_epoch(self):
        return self.eng.step_end()

    def end_epoch_async(self, sse_row, bad_cell):
        """End the step into device tensors (no host sync); returns the
        step's block ids in submission order (to decode the divergence word)."""
        self.eng.step_end_async(sse_row.data_ptr(), bad_cell.data_ptr())
        return list(self.submitted)


def _init_dist():
    import torch.distributed as dist

    if not dist.is_initialized():  # BGMF_DIST_BACKEND=gloo: tests, ranks sharing a GPU
        dist.init_process_group(backend=os.environ.get("BGMF_DIST_BACKEND", "nccl"))
    return dist


def train_blocked_distributed(d, cfg, test=None, *, early_stop: bool = True, options=None,
                              timing: bool = True):
    """Multi-GPU train_blocked (every inner schedule): every rank calls it with
    the same dataset, test set and config; rank r uses GPU LOCAL_RANK.  The
    per-step test RMSE (HoldoutEvaluator semantics, metrics.py:55-81) is
    computed where U lives: each rank evaluates the test entries of its own
    rows after the V blocks are broadcast from their holders, and the SSEs
    are all-reduced.  Returns (FactorModel on every rank, ConvergenceTrace,
    stop_reason)."""
    import torch

    dist = _init_dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    device = int(os.environ.get("BGMF_DEVICE", os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(device)
    # the engine's kernels, the NCCL V moves and the torch ops must share ONE
    # stream (NCCL orders against torch's current stream; a context created on
    # the legacy default stream would get its own non-blocking stream)
    with torch.cuda.stream(torch.cuda.Stream(device)):
        return _train_ring(d, cfg, test, early_stop, options, timing, dist, rank, world, device)


def _train_ring(d, cfg, test, early_stop, options, timing, dist, rank, world, device):
    """train_blocked_distributed's body, on the rank's training stream."""
    import torch

    from .core import ConvergenceTrace, DivergenceError, FactorModel, TraceStep
    from .kernel import divergence
    from .metrics import HoldoutEvaluator, RmseAccumulator, finalize, merge
    from .trainer import _Phases, resolve_inner_iters

    prof = _Phases() if os.environ.get("BGMF_PROFILE") and rank == 0 else None
    sched = RingSchedule(cfg.grid_i, cfg.grid_j, world)
    shard = GpuShard(d, cfg, sched, rank, device, options, _transport(world, device, dist), dist)
    closed = False
    try:
        if prof:
            torch.cuda.synchronize()
            prof.mark("shard: partition + U/V buffers")
        shard.eng.init_factors(d.n, d.m, cfg.k, cfg.seed)
        if prof:
            torch.cuda.synchronize()
            prof.mark("init_factors")
        shard.eng.prefault_factors()  # the model's host pages fault in while the epochs run
        evaluator = HoldoutEvaluator(d, test) if test is not None and len(test) > 0 else None
        if evaluator is not None:
            t = evaluator.test
            mine = shard_rows(t.rows, shard.grid.row_bounds, sched, rank)
            shard.eng.holdout_set(t.rows[mine], t.cols[mine], t.values[mine], evaluator.cold[mine],
                                  evaluator.fallback)
        nb = cfg.grid_i * cfg.grid_j
        trace = ConvergenceTrace()
        stop = "max_steps"
        total_counts = np.zeros(nb, np.int64)
        cnt = torch.tensor(shard.counts, dtype=torch.int64, device=f"cuda:{device}")
        _all_reduce(dist, cnt)
        total_counts[:] = cnt.cpu().numpy()
        from .core import AdaptiveDecreasing

        adaptive = isinstance(cfg.inner_schedule, AdaptiveDecreasing)
        hist = [0.0]
        if adaptive and int(total_counts.sum()):
            # RMSE of the initial factors over all ranks' ratings (trainer.py:98-100)
            s0 = torch.tensor([shard.eng.train_sse()], dtype=torch.float64, device=f"cuda:{device}")
            _all_reduce(dist, s0)
            hist = [math.sqrt(float(s0.item()) / int(total_counts.sum()))]
        from .core import ConvergeEachBlock

        batched = (not early_stop and evaluator is None and not adaptive
                   and not isinstance(cfg.inner_schedule, ConvergeEachBlock) and cfg.outer_steps > 1)
        pre = (_run_epochs_batched(sched, shard, rank, dist, cfg, nb, device, timing)
               if batched else None)
        for step in range(1, cfg.outer_steps + 1):
            if adaptive and step >= 2:
                prev, cur = hist[-2], hist[-1]
                ratio = (prev - cur) / prev if prev > 0 else 0.0
            else:
                ratio = 1.0
            g = resolve_inner_iters(cfg.inner_schedule, step, ratio)
            t0 = time.perf_counter()
            max_iters, capped = g, 0
            if pre is not None:  # already run: this step's results
                sse_all, order, bad_any, any_bad, g, secs = pre[step - 1]
                max_iters = g
            elif g is None:  # converge-each-block: per-block sweep counts, synchronous batches
                sse_all, order, bad_any, its, cap = _run_epoch_converge(
                    sched, shard, rank, dist, step - 1, cfg.inner_schedule.tol, cfg.alpha, cfg.beta,
                    nb, cfg.grid_j)
                agg = torch.tensor([float(its.max()) if len(its) else 0.0, float(cap)],
                                   dtype=torch.float64, device=f"cuda:{device}")
                mx = agg[:1].clone()
                _all_reduce(dist, mx, dist.ReduceOp.MAX)
                sm = agg[1:].clone()
                _all_reduce(dist, sm)
                max_iters, capped = int(mx.item()), int(sm.item())
            else:
                sse_all, order, bad_any = run_epoch(sched, shard, rank, dist, step - 1, g, cfg.alpha,
                                                    cfg.beta, nb, cfg.grid_j)
            if pre is None:
                red = torch.tensor(sse_all, device=f"cuda:{device}")
                _all_reduce(dist, red)
                sse_all = red.cpu().numpy()
                flag = torch.tensor([0 if bad_any is None else 1], device=f"cuda:{device}")
                _all_reduce(dist, flag)
                any_bad = bool(int(flag.item()))
            if any_bad or not np.all(np.isfinite(sse_all[order])):
                b = bad_any[0] if bad_any else int(next(o for o in order
                                                        if not math.isfinite(sse_all[o])))
                err = divergence(b // cfg.grid_j, b % cfg.grid_j,
                                 bad_any[1] if bad_any else int(total_counts[b]) - 1,
                                 bad_any[2] if bad_any else (g or 1) - 1)
                err.step = step
                err.partial_trace = trace
                raise err
            acc = RmseAccumulator()
            for b in order:
                acc = merge(acc, RmseAccumulator(float(sse_all[b]), int(total_counts[b])))
            train_rmse = finalize(acc)
            test_rmse = None
            if evaluator is not None:
                sync_all_v(sched, rank, shard.v_slice, dist)  # every rank needs all of V
                hs = torch.tensor([shard.eng.holdout_sse()], dtype=torch.float64,
                                  device=f"cuda:{device}")
                _all_reduce(dist, hs)
                test_rmse = math.sqrt(float(hs.item()) / len(evaluator.test))
            seconds = (secs if pre is not None else time.perf_counter() - t0) if timing else 0.0
            if shard.peer is not None:
                shard.peer.check()
            trace.append(TraceStep(step, train_rmse, test_rmse, seconds, max_iters, capped))
            hist.append(train_rmse)
            if early_stop:
                if acc.count == 0:
                    stop = "converged"
                    break
                if len(trace) >= 2 and trace.steps[-2].train_rmse - train_rmse < cfg.delta:
                    stop = "converged"
                    break
        if prof:
            torch.cuda.synchronize()
            prof.mark(f"{len(trace)} epochs")
        # gather the model: V from its holders, U row slabs from their owners
        if world > 1:
            sync_all_v(sched, rank, shard.v_slice, dist)
            for r in range(world):
                rows = sched.rows_of(r)
                if len(rows):
                    _broadcast(dist, shard.u_rows(rows), r)
        torch.cuda.synchronize()
        if prof:
            prof.mark("gather (NCCL)")
        u, v = shard.eng.get_factors()
        if prof:
            prof.mark("get_factors (D2H)")
        if shard.peer is not None:  # no rank unmaps/frees while a peer could still touch it
            torch.cuda.synchronize()
            dist.barrier()
        shard.eng.close()
        closed = True
        if prof:
            prof.mark("close")
            prof.report()
        return FactorModel(u, v), trace, stop
    except DivergenceError:
        # every rank raises together (the flag is all-reduced): peers may still
        # map this rank's V, so they leave the ring together before freeing
        if not closed and shard.peer is not None:
            torch.cuda.synchronize()
            dist.barrier()
        raise
    finally:
        if not closed:  # free the device context (and unmap peers) on any error
            if shard.peer is not None and sys.exc_info()[0] is not DivergenceError:
                shard.peer.abort()  # a local failure: do not leave peers spinning
            try:
                torch.cuda.synchronize()
            finally:
                shard.eng.close()


def bench_main(args, clock_sampler=None):
    """bench.py --gpus N under torchrun: strong scaling of the C4 epoch.
    ``clock_sampler``: bench.py's nvidia-smi sampler class (rank 0)."""
    import json

    import torch

    from . import workloads
    from .core import RatingsDataset, TrainConfig
    from .device import EngineOptions

    # NCCL / torch print banners on stdout; the driver reads ONE JSON line
    # there, so stdout is parked on stderr until that line is written
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    dist = _init_dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    device = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(device)
    w = workloads.CONFIGS[args.config]
    t_gen = time.perf_counter()
    if args.config == "C1":
        r, c, v = workloads.ml100k_standin()
    else:
        r, c, v = workloads.lowrank(w.n, w.m, args.nnz or w.nnz, seed=w.seed)
    t_gen = time.perf_counter() - t_gen
    d = RatingsDataset(w.n, w.m, r, c, v)
    nnz = len(d)
    cfg = TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, grid_i=w.grid, grid_j=w.grid,
                      seed=w.seed)
    sched = RingSchedule(w.grid, w.grid, world)
    torch.cuda.set_stream(torch.cuda.Stream(device))  # one stream: kernels + NCCL (GpuShard)
    shard = GpuShard(d, cfg, sched, rank, device, EngineOptions(timing=False),
                     _transport(world, device, dist),
                     dist)
    del r, c, v
    shard.eng.init_factors(w.n, w.m, w.k, w.seed)
    stream = shard.stream

    from dataclasses import replace

    def epochs(n):  # the trainer's batched loop: no host round trip between epochs
        _run_epochs_batched(sched, shard, rank, dist, replace(cfg, outer_steps=n),
                            w.grid * w.grid, device, False)

    epochs(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    shard.eng.set_timing(True)
    shard.eng.kernel_stats(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = None
    if rank == 0 and clock_sampler is not None:
        sampler = clock_sampler(device)
        sampler.__enter__()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    epochs(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    if sampler is not None:
        sampler.__exit__(None, None, None)
    st = shard.eng.kernel_stats(reset=True)
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{device}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # every rank's sweep launches (roofline per rank) and launch counts
    mine = torch.tensor([st["sgd_ms"], float(st["sgd_launches"]), st["sgd_alg_bytes"],
                         float(st["sse_launches"])], dtype=torch.float64,
                        device=f"cuda:{device}")
    per_rank = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(per_rank, mine)
    per_rank = [t.cpu().tolist() for t in per_rank]
    dist.barrier()
    total_ms = float(ms.item())
    shard.eng.close()
    del shard

    # e2e through the public multi-GPU API: host dataset in, host model out
    e2e = None
    if not getattr(args, "no_e2e", False):
        run_cfg = TrainConfig(k=w.k, alpha=w.alpha, beta=w.beta, grid_i=w.grid, grid_j=w.grid,
                              seed=w.seed, outer_steps=args.steps)
        train_blocked_distributed(d, TrainConfig(k=w.k, grid_i=w.grid, grid_j=w.grid,
                                                 outer_steps=1), early_stop=False)  # warm
        walls = []
        import gc

        for _ in range(5):  # median of five calls (host page state varies run to run)
            gc.collect()  # like timeit: no cyclic-GC pass inside the timed call
            gc.disable()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            train_blocked_distributed(d, run_cfg, early_stop=False)
            torch.cuda.synchronize()
            gc.enable()
            wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                                device=f"cuda:{device}")
            dist.all_reduce(wall, op=dist.ReduceOp.MAX)
            walls.append(float(wall.item()))
        t_e2e = sorted(walls)[len(walls) // 2]
        kp = (w.k + 3) // 4 * 4
        e2e = {"value": nnz * args.steps / t_e2e, "unit": "updates/s",
               "h2d_bytes_per_step": nnz * 12 / args.steps,
               "d2h_bytes_per_step": (w.n + w.m) * kp * 4 * world / args.steps,
               "what": "train_blocked_distributed(host RatingsDataset) on every rank: each "
                       "rank uploads its row shard (12 B/rating), trains, gathers the model "
                       "and downloads it as fp32 rows; median of 5 calls of the max wall "
                       "time over ranks",
               "walls_ms": [round(x * 1e3, 2) for x in walls]}
    if rank == 0:
        import json as _j

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        hbm, hbm_kind = 6650.0, "fallback (B200_PROFILING.md)"
        try:
            hbm = float(_j.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"])
            hbm_kind = "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
        launch_ms = st["sgd_ms"] / max(st["sgd_launches"], 1)
        achieved = st["sgd_alg_bytes"] / max(st["sgd_launches"], 1) / (launch_ms / 1e3) / 1e9
        ranks = []
        for r_, (sms, nl, ab, _) in enumerate(per_rank):
            lm = sms / max(nl, 1.0)
            ranks.append({"rank": r_, "avg_launch_ms": lm,
                          "achieved": ab / max(nl, 1.0) / (lm / 1e3) / 1e9 if lm > 0 else None})
        # DRAM bytes per sweep launch from the committed single-GPU ncu capture:
        # the same launch shape only at world 1 (a rank's launches hold 1/world
        # of a stratum's blocks)
        traffic = None
        if world == 1:
            try:
                cap = _j.load(open(os.path.join(root, "profiles",
                                                f"ncu_traffic_{args.config.lower()}.json")))
                traffic = next(v["dram_bytes_per_launch"] for k, v in cap.items()
                               if "sgd_fast" in k)
            except Exception:
                pass
        line = {
            "metric": "SGD rating-updates/sec (epoch)",
            "value": nnz * args.steps / (total_ms / 1e3),
            "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (workloads.lowrank)",
            "config": {"workload": w.description, "n": w.n, "m": w.m, "nnz": nnz, "k": w.k,
                       "grid": f"{w.grid}x{w.grid}",
                       "parallelism": f"U-resident/V-rotating x{world} (NCCL P2P)",
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_kind": hbm_kind,
                         "dram_frac": (traffic / (launch_ms / 1e3) / (hbm * 1e9)
                                       if traffic else None),
                         "kernel": "sgd_fast_kernel (rank 0)", "per_rank": ranks},
            "e2e": e2e, "cpu_baseline": None,
            "clocks": sampler.summary() if sampler is not None else None,
            "gpu_launches": int(sum(p[1] + p[3] for p in per_rank)),
            "gen_seconds": t_gen,
        }
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.destroy_process_group()
    sys.stdout.flush()
    os.dup2(json_fd, 1)
    os.close(json_fd)
