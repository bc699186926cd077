"""Oracle restatement of the reference sparse layer (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/lowrank/sparse.py:
  * CSR build from triples: lexsort by (row, col), duplicate rejection,
    row offsets = cumsum(bincount(rows))            (sparse.py:84-104)
  * transpose index: stable argsort of the CSR column indices, CSC offsets =
    cumsum(bincount(cols)), CSC rows = CSR rows gathered by that perm
                                                      (sparse.py:121-139)
  * Y @ X through scipy's CSR kernel (csr_matvecs), Y^T @ X through a CSR
    view of the transpose index with the values re-gathered every call
                                                      (sparse.py:153-170)
  * sampled product on the pattern in chunks of 2^18 entries
                                                      (sparse.py:19-21,173-191)
  * scaled Euclidean norm                             (sparse.py:219-228)
  * spectral-norm power iteration, tol 1e-3, <=200 steps, max of last two
                                                      (sparse.py:24-25,231-256)
"""

from __future__ import annotations

import numpy as np
import scipy.sparse

from .philox_stream import Stream

CHUNK = 1 << 18
SPECTRAL_TOL = 1e-3
SPECTRAL_STEPS = 200


class Pattern:
    """A fixed-pattern CSR matrix with a lazily-built transpose index."""

    def __init__(self, m, n, offsets, cols, vals):
        self.m, self.n = int(m), int(n)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self._rows = None
        self._t = None

    @property
    def nnz(self):
        return int(self.offsets[-1])

    def entry_rows(self):
        if self._rows is None:
            self._rows = np.repeat(np.arange(self.m, dtype=np.int64), np.diff(self.offsets))
        return self._rows

    def transpose_index(self):
        """(perm, csc_offsets, csc_rows) with perm[t] = CSR slot of CSC slot t."""
        if self._t is None:
            perm = np.argsort(self.cols, kind="stable")
            t_off = np.zeros(self.n + 1, dtype=np.int64)
            np.cumsum(np.bincount(self.cols, minlength=self.n), out=t_off[1:])
            self._t = (perm, t_off, self.entry_rows()[perm])
        return self._t

    def dense(self):
        out = np.zeros((self.m, self.n))
        out[self.entry_rows(), self.cols] = self.vals
        return out


def csr_from_triples(m, n, i, j, v) -> Pattern:
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    order = np.lexsort((j, i))
    i, j, v = i[order], j[order], v[order]
    if i.size > 1:
        same = (i[1:] == i[:-1]) & (j[1:] == j[:-1])
        if same.any():
            k = int(np.argmax(same))
            raise ValueError(f"duplicate entry at ({i[k]}, {j[k]})")
    off = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(i, minlength=m), out=off[1:])
    return Pattern(m, n, off, j, v)


def csr_times_dense(A: Pattern, X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] != A.n:
        raise ValueError(f"spmm dimension mismatch: {(A.m, A.n)} @ {X.shape}")
    view = scipy.sparse.csr_matrix((A.vals, A.cols, A.offsets), shape=(A.m, A.n), copy=False)
    return view @ X


def csr_t_times_dense(A: Pattern, X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] != A.m:
        raise ValueError(f"spmm_t dimension mismatch: {(A.m, A.n)}^T @ {X.shape}")
    perm, t_off, t_rows = A.transpose_index()
    view = scipy.sparse.csr_matrix((A.vals[perm], t_rows, t_off), shape=(A.n, A.m), copy=False)
    return view @ X


def _sampled(U, S, V, rows, cols):
    out = np.empty(rows.shape[0])
    for lo in range(0, rows.shape[0], CHUNK):
        hi = min(lo + CHUNK, rows.shape[0])
        out[lo:hi] = np.einsum("er,er->e", U[rows[lo:hi]] * S, V[cols[lo:hi]])
    return out


def sampled_product(U, S, V, A: Pattern) -> np.ndarray:
    """Entries of U diag(S) V^T at A's pattern, CSR order."""
    U, S, V = np.asarray(U), np.asarray(S), np.asarray(V)
    if U.shape[0] != A.m or V.shape[0] != A.n:
        raise ValueError("factor dims do not match pattern dims")
    if U.shape[1] != S.shape[0] or V.shape[1] != S.shape[0]:
        raise ValueError("factor rank mismatch")
    return _sampled(U, S, V, A.entry_rows(), A.cols)


def sampled_at(U, S, V, rows, cols) -> np.ndarray:
    return _sampled(np.asarray(U), np.asarray(S), np.asarray(V),
                    np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64))


def scaled_norm(x) -> float:
    x = np.asarray(x, dtype=np.float64).ravel()
    if x.size == 0:
        return 0.0
    big = np.max(np.abs(x))
    if big == 0.0:
        return 0.0
    y = x / big
    return float(big * np.sqrt(y @ y))


def spectral_estimate(A: Pattern, stream: Stream) -> float:
    if A.nnz < 1:
        raise ValueError("spectral norm estimate needs at least one stored entry")
    x = stream.normals(A.n).reshape(A.n, 1)
    x /= np.linalg.norm(x)
    last = cur = 0.0
    for _ in range(SPECTRAL_STEPS):
        z = csr_t_times_dense(A, csr_times_dense(A, x))
        lam = float(x[:, 0] @ z[:, 0])
        last, cur = cur, np.sqrt(max(lam, 0.0))
        zn = np.linalg.norm(z)
        if zn == 0.0:
            return 0.0
        x = z / zn
        if abs(cur - last) <= SPECTRAL_TOL * max(cur, 1e-300):
            break
    return max(last, cur)
