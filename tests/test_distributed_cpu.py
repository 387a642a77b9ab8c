"""Multi-GPU schedule logic on CPU: world_size 2 and 3 over gloo.

The distributed trainer's host logic (row-block ownership, the V-block moves
derived from plan_step, the per-batch exchange, plan-order SSE merge, final
model gather) is the same code the NCCL path runs (``distributed.run_epoch``,
``exchange``, ``sync_all_v``).  Here the per-block compute is the oracle (fp64,
exact), so the distributed run must be BIT-identical to the single-process
reference trainer -- any lost, stale or misrouted V block would show.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2304_13724_b200 as bm
from oracle import oracle as O
from paper_2304_13724_b200 import distributed as D
from paper_2304_13724_b200 import workloads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleShard:
    """CPU stand-in for GpuShard: this rank's ratings partitioned by the
    oracle, full-size fp64 U/V torch tensors, blocks run by oracle.sgd_sweeps."""

    def __init__(self, d, cfg, sched, rank):
        self.grid = bm.make_grid(d.n, d.m, cfg.grid_i, cfg.grid_j)
        mask = D.shard_rows(d.rows, self.grid.row_bounds, sched, rank)
        self.P = O.partition(d.rows[mask], d.cols[mask], d.values[mask], d.n, d.m, cfg.grid_i,
                             cfg.grid_j)
        u, v = O.init_factors(d.n, d.m, cfg.k, cfg.seed)
        self.U = torch.from_numpy(u.copy())
        self.V = torch.from_numpy(v.copy())
        self.J = cfg.grid_j
        self.counts = np.diff(self.P["offsets"])

    def v_slice(self, j):
        cb = self.grid.col_bounds
        return self.V[int(cb[j]):int(cb[j + 1])]

    def u_rows(self, rows):
        rb = self.grid.row_bounds
        return self.U[int(rb[rows.start]):int(rb[rows.stop])]

    def run_batch(self, blocks, g, alpha, beta):
        P, rb, cb = self.P, self.grid.row_bounds, self.grid.col_bounds
        sse = np.zeros(len(self.counts))
        ids = np.array([bi * self.J + bj for bi, bj in blocks], np.int32)
        bad = None
        U, V = self.U.numpy(), self.V.numpy()
        for pos, (bi, bj) in enumerate(blocks):
            b = bi * self.J + bj
            lo, hi = P["offsets"][b], P["offsets"][b + 1]
            us, vs = U[rb[bi]:rb[bi + 1]], V[cb[bj]:cb[bj + 1]]
            _, sa, be, bit = O.sgd_sweeps(P["rows"][lo:hi], P["cols"][lo:hi], P["values"][lo:hi],
                                          us, vs, alpha, beta, g)
            sse[b] = sa
            if be >= 0 and bad is None:
                bad = (pos, be, bit)
        return sse, bad, ids


def _worker(rank, world, port, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, cfg = case_data(case)
    sched = D.RingSchedule(cfg.grid_i, cfg.grid_j, world)
    shard = OracleShard(d, cfg, sched, rank)
    nb = cfg.grid_i * cfg.grid_j
    counts = torch.from_numpy(shard.counts.astype(np.int64))
    dist.all_reduce(counts)
    counts = counts.numpy()
    trace, moves = [], 0
    for step in range(1, cfg.outer_steps + 1):
        g = bm.resolve_inner_iters(cfg.inner_schedule, step)
        sse, order, bad = D.run_epoch(sched, shard, rank, dist, step - 1, g, cfg.alpha,
                                      cfg.beta, nb, cfg.grid_j)
        assert bad is None
        t = torch.from_numpy(sse)
        dist.all_reduce(t)
        acc = bm.RmseAccumulator()
        for b in order:
            acc = bm.merge(acc, bm.RmseAccumulator(float(t[b]), int(counts[b])))
        trace.append(bm.finalize(acc))
    # count moves a fresh schedule would make over the same steps
    s2 = D.RingSchedule(cfg.grid_i, cfg.grid_j, world)
    for step in range(cfg.outer_steps):
        for batch in s2.batches(step):
            moves += len(s2.transfers_for(batch))
    D.sync_all_v(sched, rank, shard.v_slice, dist)
    for r in range(world):
        rows = sched.rows_of(r)
        if len(rows):
            dist.broadcast(shard.u_rows(rows), src=r)
    if rank == 0:
        np.savez(os.path.join(out_dir, "dist.npz"), u=shard.U.numpy(), v=shard.V.numpy(),
                 trace=np.array(trace), moves=moves)
    dist.destroy_process_group()


def case_data(case):
    if case == "standin":
        d = workloads.ml100k_dataset()
        cfg = bm.TrainConfig(k=8, outer_steps=3, grid_i=4, grid_j=4)
    elif case == "wide":
        d = bm.gen_synthetic(bm.SyntheticSpec(40, 50, 1, 5, seed=1, density=0.5))
        cfg = bm.TrainConfig(k=6, outer_steps=3, grid_i=3, grid_j=5,
                             inner_schedule=bm.Constant(2))
    else:
        d = bm.gen_synthetic(bm.SyntheticSpec(64, 64, 1, 30, seed=0))
        cfg = bm.TrainConfig(k=10, outer_steps=4, grid_i=8, grid_j=8)
    return d, cfg


@pytest.mark.parametrize("world,case", [(2, "standin"), (3, "dense"), (2, "wide"), (4, "dense")])
def test_distributed_matches_single_process(tmp_path, world, case):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "dist.npz")
    d, cfg = case_data(case)
    u, v, tr, _ = O.train_blocked(d.n, d.m, d.rows, d.cols, d.values, k=cfg.k, alpha=cfg.alpha,
                                  beta=cfg.beta, outer_steps=cfg.outer_steps,
                                  schedule=bm.format_schedule(cfg.inner_schedule),
                                  grid_i=cfg.grid_i, grid_j=cfg.grid_j, seed=cfg.seed,
                                  early_stop=False)
    assert np.array_equal(got["u"], u)
    assert np.array_equal(got["v"], v)
    assert got["trace"].tolist() == [s["train_rmse"] for s in tr]
    assert int(got["moves"]) > 0


def test_ring_moves_match_survey_derivation():
    """P=16, G=8: within a step G blocks per batch move to g+1; at the step
    boundary all 16 blocks advance two rows = one rank."""
    s = D.RingSchedule(16, 16, 8)
    for step in range(3):
        for t, batch in enumerate(s.batches(step)):
            moves = s.transfers_for(batch)
            if step == 0 and t == 0:
                assert moves == []  # initial replicas
                continue
            if t == 0:
                assert len(moves) == 16
                assert all(m.dst == (m.src + 1) % 8 for m in moves)
            else:
                assert len(moves) == 8
                assert all(m.dst == (m.src + 1) % 8 for m in moves)
    s = D.RingSchedule(8, 8, 8)  # R = 1: every block moves every batch
    s.transfers_for(s.batches(0)[0])
    moves = s.transfers_for(s.batches(0)[1])
    assert len(moves) == 8 and all(m.dst == (m.src + 1) % 8 for m in moves)
    step_edge = D.RingSchedule(8, 8, 8)  # step boundary: +2 rows = +2 ranks
    for b in step_edge.batches(0):
        step_edge.transfers_for(b)
    moves = step_edge.transfers_for(step_edge.batches(1)[0])
    assert len(moves) == 8 and all(m.dst == (m.src + 2) % 8 for m in moves)


def test_row_ownership_covers_grid():
    for I in (1, 3, 8, 16, 17):
        for G in (1, 2, 3, 4, 8):
            s = D.RingSchedule(I, I, G)
            owned = [r for g in range(G) for r in s.rows_of(g)]
            assert owned == list(range(I))
            assert all(s.owner(r) == g for g in range(G) for r in s.rows_of(g))
            assert math.ceil(I / G) == s.R


class _FakePeerEngine:
    """Records the peer-transport calls a rank makes (no GPU)."""

    def __init__(self, rank):
        self.rank, self.calls, self._next = rank, [], 1 << 20

    def peer_alloc(self, nbytes):
        self._next += 1 << 30
        return self._next

    def peer_handle(self, base):
        return f"{self.rank}:{base}".encode()

    def peer_open(self, handle):  # mapping of rank r's base b: 10^12 (r+1) + b
        r, b = handle.split(b":")
        return 10 ** 12 * (int(r) + 1) + int(b)

    def peer_push(self, dst, src, nbytes, flag, value):
        self.calls.append(("push", dst, src, nbytes, flag, value))

    def peer_wait(self, flag, value):
        self.calls.append(("wait", flag, value))

    def peer_config(self, abort_word, timeout_s):
        self.abort_word, self.timeout_s = abort_word, timeout_s

    def peer_abort(self, peer_abort_word):
        self.calls.append(("abort", peer_abort_word))

    def peer_error(self):
        return 0


class _FakeDist:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank

    def get_world_size(self):
        return self.world

    def get_rank(self):
        return self.rank

    def all_gather_object(self, out, obj):  # every rank's handles (same bases per rank)
        for r in range(self.world):
            out[r] = tuple(h.replace(f"{self.rank}:".encode(), f"{r}:".encode()) for h in obj)

    def barrier(self):
        pass


@pytest.mark.parametrize("world,P", [(2, 8), (4, 16), (3, 7)])
def test_peer_links_sequence_and_order(world, P):
    """The peer transport's host logic over several epochs of the ring: per
    batch every push precedes every wait (a wait blocks the stream); each push
    targets the receiver's rows of that column and its flag[sender]; the k-th
    wait of receiver d on sender s expects exactly the k-th push s -> d."""
    kp, m = 8, 7 * P + 3
    cb = bm.split_bounds(m, P)
    sched = D.RingSchedule(P, P, world)
    links = []
    for r in range(world):
        eng = _FakePeerEngine(r)
        links.append(D._PeerLinks(eng, 5000, kp, cb, _FakeDist(world, r)))
    vmap = lambda d: 10 ** 12 * (d + 1) + 5000  # noqa: E731  rank d's V, mapped
    fmap = lambda d: 10 ** 12 * (d + 1) + links[d].flags  # noqa: E731
    pushes = {(s, d): [] for s in range(world) for d in range(world)}
    waits = {(s, d): [] for s in range(world) for d in range(world)}
    for step0 in range(3):
        for batch in sched.batches(step0):
            moves = sched.transfers_for(batch)
            for r, lk in enumerate(links):
                n0 = len(lk.eng.calls)
                lk.move(moves)
                kinds = [c[0] for c in lk.eng.calls[n0:]]
                assert kinds == sorted(kinds, key=lambda k: k != "push")  # pushes first
                for c in lk.eng.calls[n0:]:
                    if c[0] == "push":
                        _, dst, src, nbytes, flag, value = c
                        mv = next(mv for mv in moves if mv.src == r and
                                  dst == vmap(mv.dst) + int(cb[mv.col]) * kp * 4)
                        d = mv.dst
                        assert src - 5000 == dst - vmap(d)  # same rows, sender -> receiver
                        assert nbytes == int(cb[mv.col + 1] - cb[mv.col]) * kp * 4
                        assert flag == fmap(d) + 4 * r
                        pushes[(r, d)].append(value)
                    else:
                        _, flag, value = c
                        s = (flag - lk.flags) // 4
                        waits[(s, r)].append(value)
    for key in pushes:
        assert pushes[key] == list(range(1, len(pushes[key]) + 1))
    # bounded waits: each rank's abort word is the word after its flags; a
    # failing rank raises it in every peer's page
    for r, lk in enumerate(links):
        assert lk.eng.abort_word == lk.flags + 4 * world and lk.eng.timeout_s > 0
        n0 = len(lk.eng.calls)
        lk.abort()
        got = sorted(c[1] for c in lk.eng.calls[n0:])
        assert got == sorted(fmap(d) + 4 * world for d in range(world) if d != r)
        assert waits[key] == pushes[key]
    assert sum(len(v) for v in pushes.values()) > 0


def test_ring_transport_choice(monkeypatch):
    """Peer memory by default when every rank is on this node; torch.distributed
    for multi-node jobs (CUDA IPC is single-node) and for launchers that do not
    say how many ranks share the node; BGMF_RING_TRANSPORT wins."""
    for var in ("LOCAL_WORLD_SIZE", "BGMF_RING_TRANSPORT"):
        monkeypatch.delenv(var, raising=False)
    assert D._transport(1) == "dist"
    assert D._transport(8) == "dist"  # no LOCAL_WORLD_SIZE: not known to be one node
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert D._transport(8) == "peer"
    assert D._transport(16) == "dist"
    monkeypatch.setenv("BGMF_RING_TRANSPORT", "peer")
    assert D._transport(16) == "peer"
    monkeypatch.setenv("BGMF_RING_TRANSPORT", "nccl")
    assert D._transport(8) == "dist"
