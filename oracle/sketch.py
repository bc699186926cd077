"""Oracle restatement of the reference randomized SVDs (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/lowrank/rsvd.py:
  * params k>=1, s>=0, p>=0; width guard (k+s)[(p+1) for Krylov] <= min(m,n)
                                                      (rsvd.py:32-61)
  * rank-deficiency reroute to dense_svd(X).U when fallback is allowed,
    otherwise re-raise with an advice suffix          (rsvd.py:81-126)
  * sketch_basic = Alg. 1 (QR each product, dense SVD of Q^T A)  (rsvd.py:134-165)
  * sketch_pi    = Alg. 4 (LU in the loop, Gram-route final basis and small
    SVD, window [s, k+s))                             (rsvd.py:168-197)
  * sketch_bki   = Alg. 5 (LU blocks, QR of the concatenation, window
    [W-k, W))                                         (rsvd.py:200-231)
  * relative_fit_error = qb_error                     (rsvd.py:234-254)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .csr import Pattern, csr_t_times_dense, csr_times_dense, scaled_norm
from .dense import RankDeficient, Triplets, dense_svd, gram_svd, householder_basis, pivoted_lower
from .philox_stream import Stream, gaussian_block


@dataclass
class SketchParams:
    k: int
    p: int
    s: int = 5
    seed: int = 0

    def __post_init__(self):
        if self.k < 1:
            raise ValueError(f"rank k must be >= 1, got {self.k}")
        if self.s < 0:
            raise ValueError(f"oversampling s must be >= 0, got {self.s}")
        if self.p < 0:
            raise ValueError(f"power parameter p must be >= 0, got {self.p}")

    def guard(self, A: Pattern, krylov=False):
        w = (self.k + self.s) * ((self.p + 1) if krylov else 1)
        lim = min(A.m, A.n)
        if w > lim:
            raise ValueError(f"sketch width {w} exceeds min(m, n) = {lim}; reduce k, s or p")


@dataclass
class Basis:
    Q: np.ndarray
    provenance: str
    p: int
    fallbacks: int = 0


class _Reroute:
    def __init__(self, allowed, advice):
        self.allowed, self.advice, self.count = allowed, advice, 0

    def run(self, fn, X, dense_pick):
        try:
            return fn(X)
        except RankDeficient as exc:
            if not self.allowed:
                raise RankDeficient(f"{exc}; {self.advice}") from exc
            self.count += 1
            return dense_pick(dense_svd(X))


_U_OF = lambda t: t.U  # noqa: E731


def sketch_basic(A: Pattern, prm: SketchParams, allow_fallback=False):
    prm.guard(A)
    rr = _Reroute(allow_fallback, "matrix rank is likely below k+s, reduce k")
    omega = gaussian_block(Stream(prm.seed), A.n, prm.k + prm.s)
    Q = rr.run(householder_basis, csr_times_dense(A, omega), _U_OF)
    for _ in range(prm.p):
        G = rr.run(householder_basis, csr_t_times_dense(A, Q), _U_OF)
        Q = rr.run(householder_basis, csr_times_dense(A, G), _U_OF)
    small = dense_svd(csr_t_times_dense(A, Q).T)
    U = Q @ small.U
    k = prm.k
    return Triplets(U[:, :k], small.S[:k].copy(), small.V[:, :k], "descending"), Basis(Q, "pi", prm.p, rr.count)


def sketch_pi(A: Pattern, prm: SketchParams, allow_fallback=False):
    prm.guard(A)
    rr = _Reroute(allow_fallback, "increase s or reduce k")
    omega = gaussian_block(Stream(prm.seed), A.n, prm.k + prm.s)
    Q = csr_times_dense(A, omega)
    for step in range(prm.p + 1):
        if step == prm.p:
            Q = rr.run(lambda X: gram_svd(X).U, Q, _U_OF)
            break
        Q = rr.run(pivoted_lower, Q, _U_OF)
        Q = csr_times_dense(A, csr_t_times_dense(A, Q))
    Bt = csr_t_times_dense(A, Q)
    small = rr.run(gram_svd, Bt, lambda t: t.flipped("ascending"))
    win = slice(prm.s, prm.k + prm.s)
    res = Triplets(Q @ small.V[:, win], small.S[win].copy(), small.U[:, win], "ascending")
    return res.flipped("descending"), Basis(Q, "pi", prm.p, rr.count)


def sketch_bki(A: Pattern, prm: SketchParams, allow_fallback=False):
    prm.guard(A, krylov=True)
    rr = _Reroute(allow_fallback, "Krylov blocks are near-collinear, reduce p or use a larger matrix")
    w = prm.k + prm.s
    omega = gaussian_block(Stream(prm.seed), A.n, w)
    H = [rr.run(pivoted_lower, csr_times_dense(A, omega), _U_OF)]
    for _ in range(prm.p):
        H.append(rr.run(pivoted_lower, csr_times_dense(A, csr_t_times_dense(A, H[-1])), _U_OF))
    Q = rr.run(householder_basis, np.hstack(H), _U_OF)
    Bt = csr_t_times_dense(A, Q)
    small = rr.run(gram_svd, Bt, lambda t: t.flipped("ascending"))
    W = w * (prm.p + 1)
    win = slice(W - prm.k, W)
    res = Triplets(Q @ small.V[:, win], small.S[win].copy(), small.U[:, win], "ascending")
    return res.flipped("descending"), Basis(Q, "bki", prm.p, rr.count)


def relative_fit_error(A: Pattern, res: Triplets) -> float:
    U, S, V = res.U, res.S, res.V
    if U.shape[0] != A.m or V.shape[0] != A.n:
        raise ValueError(f"factor dims {U.shape[0]}x{V.shape[0]} do not match matrix {(A.m, A.n)}")
    if U.shape[1] != S.shape[0] or V.shape[1] != S.shape[0]:
        raise ValueError("factor rank mismatch")
    a = scaled_norm(A.vals)
    if a == 0.0:
        raise ValueError("relative error undefined for a zero matrix")
    cross = float(np.sum(csr_times_dense(A, V) * S * U))
    sq = a * a - 2.0 * cross + float(S @ S)
    return float(np.sqrt(max(sq, 0.0))) / a
