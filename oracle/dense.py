"""Oracle restatement of the reference dense layer (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/lowrank/linalg.py:
  * tolerances GRAM 1e-12 (rel. to max eigenvalue), ORTH 1e-12*||X||_F,
    LU pivot 1e-14*max|X|, dense SVD cap 2000          (linalg.py:22-31)
  * sign rule: first nonzero of each right factor column >= 0 (linalg.py:87-98)
  * householder_basis = reduced QR + |R_jj| collapse check (linalg.py:101-124)
  * pivoted_lower = GEPP P^T L via scipy lu(permute_l)  (linalg.py:127-150)
  * gram_svd = Gram (syrk), eigh of (B+B^T)/2 ascending, rank checks,
    U = A V / S, sign rule; ascending order           (linalg.py:153-202)
  * dense_svd = LAPACK gesdd, descending, size cap    (linalg.py:205-221)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

GRAM_TOL = 1e-12
ORTH_TOL = 1e-12
PIVOT_TOL = 1e-14
DENSE_CAP = 2000


class RankDeficient(Exception):
    pass


class NoConvergence(Exception):
    pass


class SizeCap(Exception):
    pass


@dataclass
class Triplets:
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    order: str

    def flipped(self, order):
        if self.order == order:
            return self
        return Triplets(self.U[:, ::-1], self.S[::-1], self.V[:, ::-1], order)

    def top(self, k):
        d = self.flipped("descending")
        return Triplets(d.U[:, :k], d.S[:k], d.V[:, :k], "descending")

    def product(self):
        return (self.U * self.S) @ self.V.T


def _as_matrix(X, what):
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or min(X.shape) < 1:
        raise ValueError(f"{what} must be 2-D with positive dims, got shape {X.shape}")
    if not np.isfinite(X).all():
        raise ValueError(f"{what} contains non-finite entries")
    return X


def sign_rule(U, V):
    for c in range(V.shape[1]):
        nz = np.flatnonzero(V[:, c])
        if nz.size and V[nz[0], c] < 0.0:
            V[:, c] *= -1.0
            U[:, c] *= -1.0


def householder_basis(X):
    X = _as_matrix(X, "orth input")
    m, n = X.shape
    if m < n:
        raise ValueError(f"orth requires m >= n, got {m}x{n}")
    fro = np.linalg.norm(X)
    if fro == 0.0:
        raise RankDeficient("cannot orthonormalize a zero matrix")
    Q, R = np.linalg.qr(X, mode="reduced")
    d = np.abs(np.diag(R))
    low = np.flatnonzero(d < ORTH_TOL * fro)
    if low.size:
        j = low[0]
        raise RankDeficient(
            f"column norm collapse at column {j} (|R[{j},{j}]| = {d[j]:.3e} < "
            f"{ORTH_TOL:.0e} * ||X||_F = {ORTH_TOL * fro:.3e})")
    return Q


def pivoted_lower(X):
    X = _as_matrix(X, "lu input")
    m, n = X.shape
    if m < n:
        raise ValueError(f"lu_pl requires m >= n, got {m}x{n}")
    big = np.max(np.abs(X))
    if big == 0.0:
        raise RankDeficient("cannot LU-factor a zero matrix")
    PL, Uf = scipy.linalg.lu(X, permute_l=True)
    piv = np.abs(np.diag(Uf))
    tol = PIVOT_TOL * big
    low = np.flatnonzero(piv < tol)
    if low.size:
        j = low[0]
        raise RankDeficient(f"zero pivot at column {j} (|pivot| = {piv[j]:.3e} < {tol:.3e})")
    return PL


def symmetric_eig(B):
    B = _as_matrix(B, "sym_eig input")
    if B.shape[0] != B.shape[1]:
        raise ValueError(f"sym_eig needs a square matrix, got {B.shape}")
    try:
        d, V = np.linalg.eigh(0.5 * (B + B.T))
    except np.linalg.LinAlgError as exc:
        raise NoConvergence(f"symmetric eigensolver did not converge: {exc}") from exc
    return V, d


def gram_svd(A):
    A = _as_matrix(A, "eig_svd input")
    m, n = A.shape
    if m < n:
        raise ValueError(f"eig_svd requires m >= n, got {m}x{n}")
    V, d = symmetric_eig(A.T @ A)
    top = d[-1]
    if top <= 0.0:
        raise RankDeficient("Gram matrix has no positive eigenvalue (zero input?)")
    low = np.flatnonzero(d <= GRAM_TOL * top)
    if low.size:
        raise RankDeficient(
            f"Gram eigenvalue {low.size} of {n} at/below rank tolerance "
            f"(index {low[0]}: {d[low[0]]:.3e} <= {GRAM_TOL:.0e} * {top:.3e})")
    S = np.sqrt(np.maximum(d, 0.0))
    U = A @ (V / S)
    sign_rule(U, V)
    return Triplets(U, S, V, "ascending")


def dense_svd(A):
    A = _as_matrix(A, "oracle_svd input")
    if min(A.shape) > DENSE_CAP:
        raise SizeCap(f"oracle SVD capped at min(m,n) <= {DENSE_CAP}, got {A.shape[0]}x{A.shape[1]}")
    U, S, Vt = np.linalg.svd(A, full_matrices=False)
    U = U.copy()
    V = Vt.T.copy()
    sign_rule(U, V)
    return Triplets(U, S, V, "descending")
