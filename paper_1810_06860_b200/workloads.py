"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The paper's MovieLens files and landscape photo are not available (and are
not reproduced); these generators produce inputs with the shapes, sizes and
value distributions BASELINE.json names.  Everything is host numpy with
recorded seeds; the observed index sets pass through `ObservationSet`, so
the CSR/CSC patterns are bit-identical for every implementation.

cfg1  1000x1000, rank-10 N(0,1) factors, 200,000 observed uniformly (seed 0)
cfg2  100000x50000, 5,000,000 uniform positions, N(0,1) values (seed 1)
cfg3  2048x2048 image shape, 50% observed.  BASELINE's wording is
      underspecified; recorded variant: 128 + U diag(255*0.9^i)
      V^T with orthonormal rank-50 U, V + N(0,1) noise, clipped to [0, 255]
                                                            (seed 3)
cfg4  138493x26744, 20,000,263 ratings: row counts Zipf(1.0) floor 20 capped
      at n; columns weighted Zipf(0.9) without replacement per row
      (exponential races for heavy rows, oversampled i.i.d. draws + dedup
      for light rows); values from a rank-20 N(0,1/sqrt(20)) product
      standardized to mean 3.5 / std 1, snapped to the 0.5 grid in [0.5,5];
      10% held out by the reference's split_observations(obs, 0.9,
      RngState(0)) (ingest.py:141-165; seed 0 = the CLI default)  (seed 4)
cfg5  1e6x2e5, 2e8 uniform positions, rank-100 product + N(0, 0.01^2) noise
      (sigma = 0.01)                                          (seed 5)
      cfg5_device: the same distribution drawn on the GPU with torch's
      generator (a different sample; ~250 s of host numpy -> seconds)
"""

from __future__ import annotations

import numpy as np


class Observations:
    """Plain container: dims, COO triples and a split tag (0 train, 1 test)."""

    def __init__(self, m, n, rows, cols, values, split=None):
        self.m, self.n = int(m), int(n)
        self.rows = np.ascontiguousarray(rows, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.split = (np.zeros(self.rows.shape[0], np.uint8) if split is None
                      else np.ascontiguousarray(split, dtype=np.uint8))

    def subset(self, tag):
        mask = self.split == tag
        return self.rows[mask], self.cols[mask], self.values[mask]


def cfg1(seed=0, m=1000, n=1000, rank=10, count=200_000):
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((m, rank))
    V = rng.standard_normal((n, rank))
    flat = rng.choice(m * n, size=count, replace=False).astype(np.int64)
    i, j = np.divmod(flat, n)
    vals = np.einsum("er,er->e", U[i], V[j])
    return Observations(m, n, i, j, vals), (U, V)


def cfg1_small(seed=20, m=200, n=150, rank=5, density=0.4):
    """A small cfg1-shaped case the oracle finishes in well under a second."""
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((m, rank))
    V = rng.standard_normal((n, rank))
    flat = rng.choice(m * n, size=int(density * m * n), replace=False).astype(np.int64)
    i, j = np.divmod(flat, n)
    vals = np.einsum("er,er->e", U[i], V[j])
    return Observations(m, n, i, j, vals), (U, V)


def uniform_sparse(m, n, nnz, seed):
    rng = np.random.default_rng(seed)
    flat = rng.choice(m * n, size=nnz, replace=False).astype(np.int64)
    i, j = np.divmod(flat, n)
    return Observations(m, n, i, j, rng.standard_normal(nnz))


def cfg2(seed=1, m=100_000, n=50_000, nnz=5_000_000):
    return uniform_sparse(m, n, nnz, seed)


def cfg3(seed=3, m=2048, n=2048, rank=50, density=0.5):
    """SURVEY.md 8(d)'s recorded variant: orthonormal rank-50 factors (QR of
    Gaussians) with singular values 255 * 0.9^i, + N(0,1) noise, a +128 gray
    offset, clipped to [0, 255].  (Without the offset half the entries clip to
    0 and SVT stalls; with it k escalates to ~316 in the first iteration,
    W ~ 1284, and the loop converges in a few iterations.)"""
    rng = np.random.default_rng(seed)
    sig = 255.0 * 0.9 ** np.arange(rank)
    U, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    V, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    X = 128.0 + (U * sig) @ V.T + rng.standard_normal((m, n))
    X = np.clip(X, 0.0, 255.0)
    flat = rng.choice(m * n, size=int(density * m * n), replace=False).astype(np.int64)
    i, j = np.divmod(flat, n)
    return Observations(m, n, i, j, X[i, j]), X


def _zipf_counts(m, n, total, s, floor):
    ranks = np.arange(1, m + 1, dtype=np.float64) ** (-s)
    lo, hi = 0.0, float(total) * 4.0
    for _ in range(200):
        C = 0.5 * (lo + hi)
        c = np.clip(np.floor(C * ranks), floor, n).astype(np.int64)
        if c.sum() > total:
            hi = C
        else:
            lo = C
    c = np.clip(np.floor(lo * ranks), floor, n).astype(np.int64)
    short = total - int(c.sum())
    room = np.flatnonzero(c < n)
    c[room[:short]] += 1
    assert int(c.sum()) == total
    return c


def split_observations(count, train_fraction, rng):
    """Train/test tags of the reference's split_observations
    (/root/reference/pkg/src/lowrank/ingest.py:141-165): n_train =
    round(fraction * count); the first n_train entries of rng.permutation(count)
    are TRAIN (0), the rest TEST (1)."""
    if not 0.0 < train_fraction < 1.0:
        raise ValueError(f"train fraction must be in (0, 1), got {train_fraction}")
    n_train = int(round(train_fraction * count))
    if n_train == 0 or n_train == count:
        raise ValueError(f"fraction {train_fraction} yields an empty split on {count} observations")
    perm = rng.permutation(count)
    split = np.ones(count, dtype=np.uint8)
    split[perm[:n_train]] = 0
    return split


def cfg4(seed=4, m=138_493, n=26_744, total=20_000_263, rank=20, train=0.9, row_cap=9_184, split_seed=0):
    """row_cap: largest per-row count (SURVEY.md 8d probe of the rating shape:
    row nnz 43 / 83 / 9,184 min/median/max); without it the literal Zipf(1)
    head fills ~60 rows completely."""
    rng = np.random.default_rng(seed)
    counts = _zipf_counts(m, min(n, row_cap), total, 1.0, 20)
    row_perm = rng.permutation(m)
    col_perm = rng.permutation(n)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-0.9)
    w /= w.sum()
    cdf = np.cumsum(w)
    rows_out, cols_out = [], []
    heavy = counts > min(1000, n // 16)
    # heavy rows: exact weighted sampling without replacement (exponential races)
    for r in np.flatnonzero(heavy):
        keys = rng.exponential(size=n) / w
        pick = np.argpartition(keys, counts[r] - 1)[: counts[r]]
        rows_out.append(np.full(counts[r], r, np.int64))
        cols_out.append(pick.astype(np.int64))
    # light rows: oversampled i.i.d. draws, dedup, keep the first c_i per row
    light = np.flatnonzero(~heavy)
    need = counts[light]
    while light.size:
        draws = need * 2 + 16
        rr = np.repeat(light, draws)
        cc = np.minimum(np.searchsorted(cdf, rng.random(rr.size), side="right"), n - 1)
        key = rr * n + cc
        _, first = np.unique(key, return_index=True)
        first.sort()
        rr, cc = rr[first], cc[first]
        # rank of each unique draw within its row (draw order)
        start = np.r_[0, np.flatnonzero(np.diff(rr)) + 1]
        rank_in_row = np.arange(rr.size) - np.repeat(start, np.diff(np.r_[start, rr.size]))
        row_need = np.zeros(m, np.int64)
        row_need[light] = need
        keep = rank_in_row < row_need[rr]
        rows_out.append(rr[keep])
        cols_out.append(cc[keep])
        got = np.bincount(rr[keep], minlength=m)
        missing = row_need - got
        light = np.flatnonzero(missing > 0)
        need = missing[light]
        if light.size:
            raise RuntimeError("cfg4 generator: oversampling left rows short; raise the draw factor")
    i = row_perm[np.concatenate(rows_out)]
    j = col_perm[np.concatenate(cols_out)]
    key = i * n + j
    uniq, idx = np.unique(key, return_index=True)
    i, j = i[idx], j[idx]
    F = rng.standard_normal((m, rank)) / np.sqrt(np.sqrt(rank))
    G = rng.standard_normal((n, rank)) / np.sqrt(np.sqrt(rank))
    x = np.einsum("er,er->e", F[i], G[j])
    x = (x - x.mean()) / x.std() + 3.5
    vals = np.clip(np.rint(x * 2.0) / 2.0, 0.5, 5.0)
    from .rng import RngState

    split = split_observations(i.size, train, RngState(split_seed))
    return Observations(m, n, i, j, vals, split)


def cfg5(seed=5, m=1_000_000, n=200_000, nnz=200_000_000, rank=100, noise=0.01):
    rng = np.random.default_rng(seed)
    keys = np.empty(0, np.int64)
    while keys.size < nnz:
        extra = rng.integers(0, m * n, size=int((nnz - keys.size) * 1.02) + 1024, dtype=np.int64)
        keys = np.unique(np.concatenate([keys, extra]))
    keys = keys[rng.permutation(keys.size)[:nnz]]
    keys.sort()
    i, j = np.divmod(keys, n)
    F = rng.standard_normal((m, rank)).astype(np.float64)
    G = rng.standard_normal((n, rank)).astype(np.float64)
    vals = np.empty(nnz)
    for lo in range(0, nnz, 1 << 22):
        hi = min(nnz, lo + (1 << 22))
        vals[lo:hi] = np.einsum("er,er->e", F[i[lo:hi]], G[j[lo:hi]])
    vals += noise * rng.standard_normal(nnz)
    return Observations(m, n, i, j, vals)


def cfg5_device(seed=5, m=1_000_000, n=200_000, nnz=200_000_000, rank=100, noise=0.01, device="cuda"):
    """cfg5's distribution sampled on the GPU (torch's Philox generator, not
    numpy's stream): uniform distinct positions (oversampled draws, unique,
    a random subset), sorted row-major; values = F_i . G_j + noise with
    F, G ~ N(0, 1).  Returns host Observations (the COO goes through
    ObservationSet like every other workload)."""
    import torch

    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    keys = torch.empty(0, dtype=torch.int64, device=dev)
    while keys.numel() < nnz:
        extra = torch.randint(0, m * n, (int((nnz - keys.numel()) * 1.02) + 1024,), generator=g, device=dev)
        keys = torch.unique(torch.cat([keys, extra]))
    keys = keys[torch.randperm(keys.numel(), generator=g, device=dev)[:nnz]]
    keys, _ = torch.sort(keys)
    i, j = keys // n, keys % n
    del keys
    F = torch.randn(m, rank, generator=g, device=dev, dtype=torch.float64)
    G = torch.randn(n, rank, generator=g, device=dev, dtype=torch.float64)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    step = 1 << 23
    for lo in range(0, nnz, step):
        hi = min(nnz, lo + step)
        vals[lo:hi] = (F[i[lo:hi]] * G[j[lo:hi]]).sum(dim=1)
    vals += noise * torch.randn(nnz, generator=g, device=dev, dtype=torch.float64)
    return Observations(m, n, i.cpu().numpy(), j.cpu().numpy(), vals.cpu().numpy())
