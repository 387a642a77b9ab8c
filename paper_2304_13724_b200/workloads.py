"""Synthetic workloads of BASELINE.json's configs C1..C5.

C1 is the reference test-suite's MovieLens-100K stand-in (reference
``tests/conftest.py:34-57``), reproduced draw-for-draw (pinned by hash in
tests/golden/golden.json).  C2..C5 use the same generative model -- train mean
3.53 + N(0, .55) user and item biases + rank-6 N(0, .6/sqrt 6) taste + N(0, .8)
noise, rounded and clipped to 1..5 -- with cells drawn without replacement by
a keyed Feistel bijection of [0, n*m) (cycle walking), which needs O(nnz)
memory instead of O(n*m) and yields the cells in scrambled (non row-major)
order, so the partitioner's sort is exercised.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import RatingsDataset

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    m: int
    nnz: int
    k: int
    grid: int
    alpha: float = 1e-4
    beta: float = 1e-2
    seed: int = 0
    description: str = ""


CONFIGS = {
    "C1": Workload("C1", 943, 1682, 100_000, 30, 4,
                   description="synthetic MovieLens-100K-shaped (943x1682, 100k), 4x4, k=30"),
    "C2": Workload("C2", 6040, 3706, 1_000_000, 32, 8,
                   description="synthetic MovieLens-1M-shaped (6040x3706, 1M), 8x8, k=32"),
    "C3": Workload("C3", 138_000, 27_000, 20_000_000, 64, 8,
                   description="synthetic MovieLens-20M-shaped (138k x 27k, 20M), 8x8, k=64"),
    "C4": Workload("C4", 480_000, 17_800, 100_000_000, 128, 16,
                   description="synthetic Netflix-shaped (480k x 17.8k, 100M), 16x16, k=128"),
    "C5": Workload("C5", 10_000_000, 1_000_000, 2_000_000_000, 128, 64,
                   description="synthetic 10M x 1M, 2B ratings, k=128, out-of-core"),
    # C4 with skew: user and item popularity follow shifted power laws (the
    # real MovieLens / Netflix data the paper trains on are heavy-tailed,
    # PAPER.md:252,294); same shape, grid, k and rating model as C4
    "C4Z": Workload("C4Z", 480_000, 17_800, 100_000_000, 128, 16,
                    description="synthetic Netflix-shaped with Zipf users and items "
                                "(480k x 17.8k, 100M), 16x16, k=128"),
}


def ml100k_standin():
    """(rows, cols, values) of the reference's C1 stand-in generator."""
    g = np.random.default_rng(100_000)
    n_users, n_items, n_ratings, f = 943, 1682, 100_000, 6
    b_user = g.normal(0.0, 0.55, n_users)
    b_item = g.normal(0.0, 0.55, n_items)
    taste_u = g.normal(0.0, 0.6 / np.sqrt(f), (n_users, f))
    taste_v = g.normal(0.0, 0.6 / np.sqrt(f), (n_items, f))
    flat = g.choice(n_users * n_items, size=n_ratings, replace=False)
    rows, cols = np.divmod(flat, n_items)
    raw = (3.53 + b_user[rows] + b_item[cols]
           + np.einsum("ij,ij->i", taste_u[rows], taste_v[cols])
           + g.normal(0.0, 0.8, n_ratings))
    return rows, cols, np.clip(np.rint(raw), 1, 5).astype(np.int64)


def ml100k_dataset() -> RatingsDataset:
    r, c, v = ml100k_standin()
    return RatingsDataset(943, 1682, r, c, v)


def _mix(x: np.ndarray, key: np.uint64) -> np.ndarray:
    """splitmix64-style finaliser of (x ^ key); uint64 wraparound."""
    with np.errstate(over="ignore"):
        z = x ^ key
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def feistel_cells(total: int, count: int, seed: int, start: int = 0) -> np.ndarray:
    """perm(start .. start+count) for a keyed bijection perm of [0, total)."""
    bits = max(2, int(total - 1).bit_length())
    lo_bits = bits // 2
    hi_bits = bits - lo_bits
    lo_mask = np.uint64((1 << lo_bits) - 1)
    hi_mask = np.uint64((1 << hi_bits) - 1)
    keys = [np.uint64((seed * 0x9E3779B97F4A7C15 + r * 0xD1B54A32D192ED03 + 1) & (2**64 - 1))
            for r in range(4)]

    def perm(x: np.ndarray) -> np.ndarray:
        hi = x >> np.uint64(lo_bits)
        lo = x & lo_mask
        # unbalanced Feistel: alternate which half is mixed; each round is invertible
        for r in range(4):
            if r % 2 == 0:
                hi = (hi ^ _mix(lo, keys[r])) & hi_mask
            else:
                lo = (lo ^ _mix(hi, keys[r])) & lo_mask
        return (hi << np.uint64(lo_bits)) | lo

    x = np.arange(start, start + count, dtype=np.uint64)
    y = perm(x)
    t = np.uint64(total)
    pending = np.flatnonzero(y >= t)
    while pending.size:  # cycle walking keeps the map a bijection of [0, total)
        y[pending] = perm(y[pending])
        pending = pending[y[pending] >= t]
    return y.astype(np.int64)


def lowrank(n: int, m: int, nnz: int, seed: int = 0, chunk: int = 1 << 24):
    """(rows int64, cols int64, values float64) of the C2..C5 generator."""
    g = np.random.default_rng(seed)
    f = 6
    b_user = g.normal(0.0, 0.55, n)
    b_item = g.normal(0.0, 0.55, m)
    taste_u = g.normal(0.0, 0.6 / np.sqrt(f), (n, f)).astype(np.float32)
    taste_v = g.normal(0.0, 0.6 / np.sqrt(f), (m, f)).astype(np.float32)
    rows = np.empty(nnz, np.int64)
    cols = np.empty(nnz, np.int64)
    vals = np.empty(nnz, np.float64)
    for s in range(0, nnz, chunk):
        e = min(nnz, s + chunk)
        cells = feistel_cells(n * m, e - s, seed, start=s)
        r, c = np.divmod(cells, m)
        raw = (3.53 + b_user[r] + b_item[c]
               + np.einsum("ij,ij->i", taste_u[r], taste_v[c]).astype(np.float64)
               + g.normal(0.0, 0.8, e - s))
        rows[s:e], cols[s:e] = r, c
        vals[s:e] = np.clip(np.rint(raw), 1, 5)
    return rows, cols, vals


def _power_cdf(count: int, shift: float, expo: float) -> np.ndarray:
    w = (np.arange(count, dtype=np.float64) + 1.0 + shift) ** -expo
    cdf = np.cumsum(w)
    return cdf / cdf[-1]


def zipf_cells(n: int, m: int, nnz: int, seed: int = 0, user_shift: float = 500.0,
               user_expo: float = 0.9, item_shift: float = 50.0,
               item_expo: float = 1.0, device: str | None = None) -> np.ndarray:
    """nnz distinct cells of an n x m matrix, users and items drawn with
    probability ~ (rank + shift)^-expo (ranks scattered over the ids by a
    seeded permutation, so heavy users and hot items land in every block).
    Defaults: the hottest item gets ~0.3% of the ratings (~half the users,
    like Netflix's), the heaviest users rate most of the items; cells in
    scrambled order.  Drawn with torch's generator on `device` (default
    cuda:0 when present: 100 M distinct cells in seconds; the CPU stream
    differs, so a dataset is only comparable within one device kind)."""
    import torch

    dev = device or ("cuda:0" if torch.cuda.is_available() else "cpu")
    g = torch.Generator(device=dev)
    g.manual_seed(seed * 1_000_003 + 0x5A1F)

    def cdf(count, shift, expo):
        w = (torch.arange(count, device=dev, dtype=torch.float64) + 1.0 + shift) ** -expo
        c = torch.cumsum(w, 0)
        return c / c[-1]

    ucdf, icdf = cdf(n, user_shift, user_expo), cdf(m, item_shift, item_expo)
    uperm = torch.randperm(n, generator=g, device=dev)
    iperm = torch.randperm(m, generator=g, device=dev)
    have = torch.empty(0, dtype=torch.int64, device=dev)
    while have.numel() < nnz:
        draw = int((nnz - have.numel()) * 1.15) + 1024
        u = uperm[torch.searchsorted(ucdf, torch.rand(draw, generator=g, device=dev,
                                                      dtype=torch.float64)).clamp_(max=n - 1)]
        i = iperm[torch.searchsorted(icdf, torch.rand(draw, generator=g, device=dev,
                                                      dtype=torch.float64)).clamp_(max=m - 1)]
        have = torch.unique(torch.cat([have, u * m + i]))
        del u, i
    keep = torch.randperm(have.numel(), generator=g, device=dev)[:nnz]
    out = have[keep].cpu().numpy()
    del have, keep
    return out


def zipf_lowrank(n: int, m: int, nnz: int, seed: int = 0, chunk: int = 1 << 24):
    """(rows, cols, values) of C4Z: zipf_cells with lowrank's rating model."""
    g = np.random.default_rng(seed)
    f = 6
    b_user = g.normal(0.0, 0.55, n)
    b_item = g.normal(0.0, 0.55, m)
    taste_u = g.normal(0.0, 0.6 / np.sqrt(f), (n, f)).astype(np.float32)
    taste_v = g.normal(0.0, 0.6 / np.sqrt(f), (m, f)).astype(np.float32)
    cells = zipf_cells(n, m, nnz, seed)
    rows, cols = np.divmod(cells, m)
    vals = np.empty(nnz, np.float64)
    for s in range(0, nnz, chunk):
        e = min(nnz, s + chunk)
        r, c = rows[s:e], cols[s:e]
        raw = (3.53 + b_user[r] + b_item[c]
               + np.einsum("ij,ij->i", taste_u[r], taste_v[c]).astype(np.float64)
               + g.normal(0.0, 0.8, e - s))
        vals[s:e] = np.clip(np.rint(raw), 1, 5)
    return rows, cols, vals


def generate(name: str, nnz: int | None = None):
    """(rows, cols, values) of workload `name` (C1 .. C5, C4Z)."""
    w = CONFIGS[name]
    if name == "C1":
        r, c, v = ml100k_standin()
        return r, c, v.astype(np.float64)
    if name == "C4Z":
        return zipf_lowrank(w.n, w.m, nnz or w.nnz, w.seed)
    return lowrank(w.n, w.m, nnz or w.nnz, w.seed)


def dataset(name: str, nnz: int | None = None) -> RatingsDataset:
    w = CONFIGS[name]
    if name == "C1":
        return ml100k_dataset()
    r, c, v = lowrank(w.n, w.m, nnz or w.nnz, w.seed)
    return RatingsDataset(w.n, w.m, r, c, v)
