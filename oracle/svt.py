"""Oracle restatement of the reference SVT engine (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/lowrank/completion.py:
  * config defaults and validation                  (completion.py:44-88)
  * shrink: r = #{S > tau}, S[:r] - tau              (completion.py:157-167)
  * power rule: increase -> p+1, streak 0; else streak+1, at 10 -> p-1 (>= p_min)
                                                      (completion.py:181-197)
  * recycling: restart from cached Q (window [W-k, W)) or rotate cached U
                                                      (completion.py:200-245)
  * inner SVD routing: recycle gate (strategy, i >= i_reuse, q < q_reuse,
    width fits), stale -> fresh; width clamp budget = min_dim//(k+s) - 1,
    dense when < 1; p_eff = max(1, min(p, budget)); seed = root.derive(calls)
                                                      (completion.py:248-310)
  * the loop: tau = 5n, delta = 1.2mn/nnz, c = ceil(tau/(delta*||P(M)||_2)),
    Y0 = c*delta*P(M); per iteration k = r_prev+1, escalate by l until
    S[k-1] <= tau or k = min(m,n); shrink; residual; stop before update;
    Y += step*(M - X) on the pattern; power rule for the BKI backend only
                                                      (completion.py:313-406)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .csr import Pattern, csr_from_triples, csr_t_times_dense, sampled_product, scaled_norm, spectral_estimate
from .dense import RankDeficient, Triplets, dense_svd, gram_svd
from .philox_stream import Stream
from .sketch import SketchParams, sketch_bki


@dataclass
class SvtConfig:
    tau: Optional[float] = None
    delta: Optional[float] = None
    l: int = 5
    epsilon: float = 0.05
    i_max: int = 500
    i_reuse: int = 100
    q_reuse: int = 10
    strategy: str = "none"
    p0: int = 3
    p_min: int = 1
    s: int = 5
    seed: int = 0
    delta_decay: bool = False


@dataclass
class _Loop:
    Y: Pattern
    r_prev: int = 0
    p: int = 3
    q: int = 0
    streak: int = 0
    history: list = field(default_factory=list)
    cached_q: Optional[object] = None
    cached_u: Optional[np.ndarray] = None
    iteration: int = 0
    dense_cache: Optional[Triplets] = None
    calls: int = 0
    p_min: int = 1
    root: Optional[Stream] = None


def run_power_rule(loop, err):
    if loop.history and err > loop.history[-1]:
        loop.p += 1
        loop.streak = 0
    else:
        loop.streak += 1
        if loop.streak >= 10:
            loop.p = max(loop.p_min, loop.p - 1)
            loop.streak = 0
    loop.history.append(err)
    return loop.p


def restart_from_q(basis, Y: Pattern, k):
    W = basis.Q.shape[1]
    if k > W:
        raise ValueError(f"requested rank {k} exceeds cached subspace width {W}")
    if k == 0:
        return Triplets(np.zeros((basis.Q.shape[0], 0)), np.zeros(0), np.zeros((Y.n, 0)), "descending")
    small = gram_svd(csr_t_times_dense(Y, basis.Q))
    win = slice(W - k, W)
    return Triplets(basis.Q @ small.V[:, win], small.S[win].copy(), small.U[:, win], "ascending").flipped("descending")


def rotate_u(U_prev, Y: Pattern):
    k = U_prev.shape[1]
    if k == 0:
        return Triplets(np.zeros((U_prev.shape[0], 0)), np.zeros(0), np.zeros((Y.n, 0)), "descending")
    try:
        small = gram_svd(csr_t_times_dense(Y, U_prev))
    except RankDeficient as exc:
        raise RankDeficient(f"projection onto cached U lost rank ({exc}); refresh the subspace") from exc
    return Triplets(U_prev @ small.V, small.S.copy(), small.U.copy(), "ascending").flipped("descending")


def _inner(loop, cfg, backend, strategy, k, events):
    Y = loop.Y
    lo = min(Y.m, Y.n)
    loop.calls += 1
    if backend == "oracle":
        if loop.dense_cache is None:
            loop.dense_cache = dense_svd(Y.dense())
        return loop.dense_cache.top(k), "oracle"
    fits = False
    if strategy == "reuse-q":
        fits = loop.cached_q is not None and k <= loop.cached_q.Q.shape[1]
    elif strategy == "reuse-u":
        fits = loop.cached_u is not None and k <= loop.cached_u.shape[1]
    if strategy != "none" and loop.iteration >= cfg.i_reuse and loop.q < cfg.q_reuse and fits:
        try:
            if strategy == "reuse-q":
                res, src = restart_from_q(loop.cached_q, Y, k), "recycle-q"
            else:
                res, src = rotate_u(loop.cached_u, Y), "recycle-u"
            loop.q += 1
            if strategy == "reuse-u":
                loop.cached_u = res.U
            return res, src
        except RankDeficient:
            events.append(f"i={loop.iteration} k={k}: stale subspace, refreshing")
    budget = lo // (k + cfg.s) - 1
    if budget < 1:
        events.append(f"i={loop.iteration} k={k}: BKI width clamp, dense SVD")
        res = dense_svd(Y.dense()).top(k)
        loop.q = 0
        if strategy == "reuse-u":
            loop.cached_u = res.U
        return res, "oracle"
    prm = SketchParams(k=k, p=max(1, min(loop.p, budget)), s=cfg.s, seed=loop.root.derive(loop.calls).seed)
    res, basis = sketch_bki(Y, prm, allow_fallback=True)
    loop.q = 0
    if basis.fallbacks:
        events.append(f"i={loop.iteration} k={k}: {basis.fallbacks} dense fallback(s) in BKI")
    if strategy == "reuse-q":
        loop.cached_q = basis
    if strategy == "reuse-u":
        loop.cached_u = res.U
    return res, "bki"


@dataclass
class Outcome:
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    rank: int
    iterations: int
    converged: bool
    residual: float
    trace: list
    events: list
    c: int
    norm2: float
    hard_stops: int = 0


def complete(m, n, rows, cols, vals, cfg: SvtConfig, backend="rsvd-bki", strategy=None):
    """SVT on the observed triples (train split only). strategy None -> cfg.strategy."""
    strategy = cfg.strategy if strategy is None else strategy
    phi = csr_from_triples(m, n, rows, cols, vals)
    if phi.nnz == 0:
        raise ValueError("no observed entries to complete from")
    lo = min(m, n)
    mv = phi.vals.copy()
    mnorm = scaled_norm(mv)
    if mnorm == 0.0:
        raise ValueError("observed entries are all zero; nothing to recover")
    tau = cfg.tau if cfg.tau is not None else 5.0 * n
    delta = cfg.delta if cfg.delta is not None else 1.2 * m * n / phi.nnz
    root = Stream(cfg.seed)
    norm2 = spectral_estimate(phi, root.derive(1))
    c = math.ceil(tau / (delta * norm2))
    Y = Pattern(m, n, phi.offsets, phi.cols, c * delta * mv)
    loop = _Loop(Y=Y, p=cfg.p0, p_min=cfg.p_min, root=root)
    trace, events = [], []
    hard = 0
    conv = False
    out = (np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)), 0)
    resid = float("inf")
    for it in range(1, cfg.i_max + 1):
        loop.iteration = it
        loop.dense_cache = None
        k = loop.r_prev + 1
        while True:
            ke = min(k, lo)
            res, src = _inner(loop, cfg, backend, strategy, ke, events)
            if res.S[ke - 1] <= tau:
                break
            if ke == lo:
                hard += 1
                events.append(f"i={it}: rank escalation hit min(m, n) = {lo}")
                break
            k += cfg.l
        r = int(np.count_nonzero(res.S > tau))
        Us, Ss, Vs = res.U[:, :r].copy(), res.S[:r] - tau, res.V[:, :r].copy()
        loop.r_prev = r
        out = (Us, Ss, Vs, r)
        x = sampled_product(Us, Ss, Vs, phi) if r > 0 else np.zeros(phi.nnz)
        resid = scaled_norm(x - mv) / mnorm
        trace.append((it, ke, r, loop.p, loop.q, resid, src))
        if resid < cfg.epsilon:
            conv = True
            break
        step = delta * (0.999 ** it) if cfg.delta_decay else delta
        Y.vals += step * (mv - x)
        if backend == "rsvd-bki":
            run_power_rule(loop, resid)
    Us, Ss, Vs, r = out
    return Outcome(Us, Ss, Vs, r, len(trace), conv, resid, trace, events, c, norm2, hard)
