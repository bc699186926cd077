"""Host (numpy) kernel set for the sharded engine -- TEST INFRASTRUCTURE ONLY.

paper_1810_06860_b200.shards.ShardedEngine takes its per-rank operations
from a kernel set; the product passes shards.DeviceKernels (the sm_100a
library).  The world-size-2 gloo tests in tests/test_shards_gloo.py inject
this numpy restatement instead, built on the oracle (oracle/), so the
sharding choreography -- partition, allgathers, allreduces, replicated
solves, rank agreement -- runs on a CPU box.  Tensors are torch CPU float64
(what gloo moves); arithmetic is the oracle's.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import torch

import oracle
from oracle import csr as ocsr
from oracle import dense as odense
from paper_1810_06860_b200.errors import NumericalError, RankDeficiencyError, SizeCapError


def _np(t):
    return t.numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


class HostPower:
    """oracle.spectral_estimate's state machine, one update per A^T A x."""

    def __init__(self, x0):
        x = np.asarray(x0, dtype=np.float64).reshape(-1, 1)
        self.x = torch.from_numpy(x / np.linalg.norm(x))
        self.last = self.cur = 0.0
        self._done = self._zero = False

    def update(self, z):
        if self._done:
            return
        x, z = _np(self.x), _np(z)
        lam = float(x[:, 0] @ z[:, 0])
        self.last, self.cur = self.cur, float(np.sqrt(max(lam, 0.0)))
        zn = float(np.linalg.norm(z))
        if zn == 0.0:
            self._zero = self._done = True
            return
        self.x = torch.from_numpy(z / zn)
        if abs(self.cur - self.last) <= ocsr.SPECTRAL_TOL * max(self.cur, 1e-300):
            self._done = True

    def done(self):
        return self._done

    def result(self):
        return 0.0 if self._zero else max(self.last, self.cur)


class HostKernels:
    def empty(self, rows, cols):
        return torch.zeros((rows, cols), dtype=torch.float64)

    def vector(self, values):
        return torch.from_numpy(np.array(values, dtype=np.float64).ravel())

    def from_host(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def to_host(self, t):
        return _np(t).copy()

    def copy(self, src, dst):
        dst.copy_(src)

    # sparse blocks (oracle Pattern)
    def block(self, rows, cols, indptr, indices, data, prep=None, slot=0):
        return ocsr.Pattern(rows, cols, indptr, indices, np.array(data, dtype=np.float64))

    def block_like(self, A, data):
        B = ocsr.Pattern(A.m, A.n, A.offsets, A.cols, np.array(data, dtype=np.float64))
        B._rows, B._t = A._rows, A._t
        return B

    def scaled_block(self, A, scale):
        return self.block_like(A, float(scale) * A.vals)

    def host_values(self, A):
        return A.vals

    def values(self, A):
        return torch.from_numpy(A.vals.copy())

    def densify(self, A):
        return A.dense()

    def spmm(self, A, X, out):
        out.copy_(torch.from_numpy(np.asarray(ocsr.csr_times_dense(A, _np(X)))))
        return out

    def spmm_t(self, A, X, out):
        out.copy_(torch.from_numpy(np.asarray(ocsr.csr_t_times_dense(A, _np(X)))))
        return out

    def _x(self, A, U, S, V, r):
        if r == 0:
            return np.zeros(A.nnz)
        return ocsr.sampled_product(_np(U), _np(S), _np(V), A)

    def svt_step(self, A, m_vals, U, S, V, r, step):
        x = self._x(A, U, S, V, r)
        m = _np(m_vals)
        d = x - m
        A.vals += step * (m - x)
        return torch.tensor([float(d @ d), float(np.max(np.abs(d))) if d.size else 0.0], dtype=torch.float64)

    def project(self, A, U, S, V, r):
        return torch.from_numpy(self._x(A, U, S, V, r))

    def stats(self, x):
        a = _np(x).ravel()
        fin = np.isfinite(a)
        return torch.tensor([float(a @ a) if a.size else 0.0, float(np.max(np.abs(a))) if a.size else 0.0,
                             float(np.count_nonzero(~fin))], dtype=torch.float64)

    def scaled_stats(self, x, big):
        return self.stats(torch.from_numpy(_np(x) / big))

    def power(self, x0):
        return HostPower(x0)

    # dense
    def gram(self, X):
        a = _np(X)
        return torch.from_numpy(a.T @ a)

    def matmul(self, A, B, b_upper=False):
        b = _np(B)
        return torch.from_numpy(_np(A) @ (np.triu(b) if b_upper else b))

    def potrf_inv(self, G, shift=0.0):
        g = _np(G).copy()
        if shift:
            g[np.diag_indices_from(g)] += shift
        c, info = scipy.linalg.lapack.dpotrf(g, lower=0, clean=1)
        if info:
            return int(info), None
        G.copy_(torch.from_numpy(c))
        rinv = scipy.linalg.solve_triangular(c, np.eye(c.shape[0]), lower=False)
        return 0, torch.from_numpy(rinv)

    def diag(self, G):
        return np.diag(_np(G)).copy()

    def sym_eig(self, G):
        try:
            V, d = odense.symmetric_eig(_np(G))
        except odense.NoConvergence as exc:
            raise NumericalError(str(exc)) from exc
        return torch.from_numpy(np.ascontiguousarray(V)), np.asarray(d)

    def fix_signs(self, V):
        v = _np(V)
        for c in range(v.shape[1]):
            nz = np.flatnonzero(v[:, c])
            if nz.size and v[nz[0], c] < 0.0:
                v[:, c] *= -1.0

    def select_columns(self, V, cols, S=None):
        v = _np(V)[:, np.asarray(cols)]
        if S is not None:
            v = v / np.asarray(S)[np.asarray(cols)]
        return torch.from_numpy(np.ascontiguousarray(v))

    def lu_pl(self, X):
        try:
            PL = odense.pivoted_lower(_np(X))
        except odense.RankDeficient as exc:
            raise RankDeficiencyError(str(exc)) from exc
        X.copy_(torch.from_numpy(PL))
        return X

    def lu_pl_async(self, X, status):
        """The speculative route's LU: status[0] = -1 when the pivots hold,
        else the careful path is replayed (lr_lu_pl_async_f64's contract)."""
        try:
            PL = odense.pivoted_lower(_np(X))
        except odense.RankDeficient:
            status[0] = 0.0
            return
        X.copy_(torch.from_numpy(PL))
        status[0] = -1.0

    def gaussian(self, seed, rows, cols):
        return torch.from_numpy(oracle.gaussian_block(oracle.Stream(seed), rows, cols))

    def dense_svd(self, X):
        try:
            t = odense.dense_svd(_np(X))
        except odense.SizeCap as exc:
            raise SizeCapError(str(exc)) from exc
        return torch.from_numpy(t.U), np.asarray(t.S), torch.from_numpy(t.V)
