"""Dense building blocks of the randomized SVDs, on the device.

Drop-in for /root/reference/pkg/src/lowrank/linalg.py (same names, result
types, orders, tolerances and error messages).  The LAPACK calls of the
reference are replaced by the native library:

  orth      Householder QR (dgeqrf/dorgqr)  -> CholeskyQR2 on DMMA Grams,
            shifted CholeskyQR3 when the first Cholesky breaks down; the
            |R_jj| collapse test uses R = R2 R1 (R3 R2 R1), whose diagonal is
            the unique positive-diagonal R of X = QR       (linalg.py:101-124)
  lu_pl     dgetrf + P L                    -> cooperative GEPP kernel
                                                            (linalg.py:127-150)
  sym_eig   dsyevd                          -> Householder tridiagonalization +
            bisection + inverse iteration (lr_syevd_f64); the parallel
            block-Jacobi solver lr_syevj_f64 is opt-in (EIG_METHOD)
                                                            (linalg.py:153-169)
  eig_svd   dsyrk + dsyevd + dgemm          -> DMMA syrk + syevd + DMMA gemm
                                                            (linalg.py:172-202)
  oracle_svd dgesdd (dense, capped)         -> Gram-preconditioned one-sided Jacobi (abs. accuracy)
            by CholeskyQR2 (orthonormal completion for null directions)
                                                            (linalg.py:205-221)

Public functions take and return numpy arrays (CUDA tensors pass through
as tensors); the `*_dev` variants keep everything on the device and are what
rsvd.py / completion.py call.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, device
from .errors import NumericalError, RankDeficiencyError, SizeCapError

GRAM_RANK_TOL = 1e-12
ORTH_RANK_TOL = 1e-12
LU_PIVOT_TOL = 1e-14
ORACLE_SVD_CAP = 2000
JACOBI_MAX_SWEEPS = 60
# "syevd": tridiagonalization + bisection + inverse iteration (default);
# "syevj": parallel block Jacobi (relative accuracy, slower at large n)
EIG_METHOD = "syevd"
_U_ROUND = 2.0 ** -53


@dataclass
class SvdResult:
    """Economic SVD triple with an explicit order ("ascending"/"descending")."""

    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    order: str

    @property
    def rank(self) -> int:
        return self.S.shape[0]

    def descending(self) -> "SvdResult":
        if self.order == "descending":
            return self
        return SvdResult(self.U[:, ::-1], self.S[::-1], self.V[:, ::-1], "descending")

    def ascending(self) -> "SvdResult":
        if self.order == "ascending":
            return self
        return SvdResult(self.U[:, ::-1], self.S[::-1], self.V[:, ::-1], "ascending")

    def truncate(self, k: int) -> "SvdResult":
        d = self.descending()
        return SvdResult(d.U[:, :k], d.S[:k], d.V[:, :k], "descending")

    def reconstruct(self) -> np.ndarray:
        return (self.U * self.S) @ self.V.T


@dataclass
class DevSvd:
    """Device triple, always descending; S_host mirrors S for host decisions."""

    U: object
    S: object
    V: object
    S_host: np.ndarray
    V_pending: object = None  # device.PendingHost of V started before U was lifted

    def to_host(self) -> SvdResult:
        V = self.V_pending.result() if self.V_pending is not None else device.to_host(self.V)
        return SvdResult(device.to_host(self.U), self.S_host.copy(), V, "descending")


# ------------------------------------------------------------------ helpers

def _st():
    return device.stream()


def _gemm(transA, M, N, K, alpha, A, B, beta, C, flags=0, work_name="gemm_work"):
    need = int(_native.load().lr_gemm_workspace_doubles(transA, M, N, K, flags))
    work = device.arena().get(work_name, need) if need else None
    _native.call("lr_gemm_f64", transA, M, N, K, alpha, device.ptr(A), device.ld(A), device.ptr(B),
                 device.ld(B), beta, device.ptr(C), device.ld(C), flags, device.ptr(work),
                 int(work.numel()) if work is not None else 0, _st(),
                 meta={"M": M, "N": N, "K": K, "transA": transA, "flags": flags})
    return C


def gram_dev(A, out=None):
    """A^T A (exactly symmetric, upper tiles mirrored)."""
    rows, n = A.shape
    if out is None:
        out = device.empty(n, n)
    return _gemm(1, n, n, rows, 1.0, A, A, 0.0, out, _native.LR_GEMM_SYRK_UPPER)


def gram_tf32x3_dev(A32, out=None):
    """A^T A of an fp32 block on the tcgen05 tensor cores (3xTF32, fp64
    result, exactly symmetric): the fp32 mode's eigSVD Gram."""
    rows, n = A32.shape
    if out is None:
        out = device.empty(n, n)
    nf = int(_native.load().lr_gram_tf32x3_workspace_floats(rows, n))
    work = device.arena().get("gram_tf32x3", (nf + 1) // 2)
    _native.call("lr_gram_tf32x3", device.ptr(A32), device.ld(A32), rows, n, device.ptr(out), device.ld(out),
                 device.ptr(work), 2 * int(work.numel()), _st())
    return out


def matmul_dev(A, B, out=None, b_upper=False):
    """A (M x K) @ B (K x N)."""
    M, K = A.shape
    N = B.shape[1]
    if out is None:
        out = device.empty(M, N)
    return _gemm(0, M, N, K, 1.0, A, B, 0.0, out, _native.LR_GEMM_B_UPPER if b_upper else 0)


def matmul_tn_dev(A, B, out=None):
    """A^T (M x K) @ B (K x N), A is K x M."""
    K, M = A.shape
    N = B.shape[1]
    if out is None:
        out = device.empty(M, N)
    return _gemm(1, M, N, K, 1.0, A, B, 0.0, out, 0, "gemm_work_tn")


def stats_dev(X):
    """(sum of squares, max|x|, #non-finite) of a device block, one sync."""
    rows, cols = X.shape
    if rows * cols == 0:
        return 0.0, 0.0, 0
    part = device.arena().get("stats_partial", _native.load().lr_stats_partials() + 8)
    out = device.vector(3)
    _native.call("lr_block_stats_f64", device.ptr(X), rows, cols, device.ld(X), device.ptr(part),
                 device.ptr(out), _st())
    h = device.to_host(out)
    return float(h[0]), float(h[1]), int(h[2])


def _check_dev(X, name):
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise ValueError(f"{name} must be 2-D with positive dims, got shape {tuple(X.shape)}")
    s = stats_dev(X)
    if s[2]:
        raise ValueError(f"{name} contains non-finite entries")
    return s


def _fro_from_stats(s, X):
    sumsq, big = s[0], s[1]
    if big == 0.0:
        return 0.0
    if np.isfinite(sumsq) and 1e-150 < big < 1e150:
        return float(np.sqrt(sumsq))
    from .sparse import frobenius_dev

    return frobenius_dev(X)


def _diag_host(R, n):
    d = device.vector(n)
    _native.call("lr_diag_f64", device.ptr(R), device.ld(R), n, device.ptr(d), _st())
    return device.to_host(d)


def potrf_inv_dev(G, shift=0.0):
    """In place upper Cholesky of G (+ shift I); returns (info, Rinv)."""
    n = G.shape[0]
    Rinv = device.empty(n, n)
    work = device.arena().get("potrf_work", int(_native.load().lr_potrf_workspace_doubles(n)))
    info = ctypes.c_int(0)
    _native.call("lr_potrf_inv_f64", n, device.ptr(G), device.ld(G), float(shift), device.ptr(Rinv),
                 device.ld(Rinv), device.ptr(work), ctypes.byref(info), _st())
    return int(info.value), Rinv


# --------------------------------------------------------------------- orth

class LazyQ:
    """Q = base @ Rinv (Rinv upper triangular) kept unformed: the last
    CholeskyQR pass of `orth` for callers that only need Y^T Q and Q V
    (rsvd_bki's projection: (Y^T base) Rinv and base (Rinv V) -- one m x W x W
    pass fewer).  `materialize()` forms Q once, on demand."""

    def __init__(self, base, Rinv):
        self.base, self.Rinv = base, Rinv
        self.R1inv = None  # base = X R1inv when the speculative route built it (orth_speculative_dev)
        self.T_all = None  # Y^T X, when the caller kept it (rsvd._krylov_orth)
        self._Q = None

    @property
    def shape(self):
        return (int(self.base.shape[0]), int(self.Rinv.shape[1]))

    def materialize(self):
        if self._Q is None:
            self._Q = matmul_dev(self.base, self.Rinv, b_upper=True)
        return self._Q


def _cholqr_pass(X, shift=0.0, G=None, lazy=False):
    """One CholeskyQR pass: returns (info, Q, diag(R)); G = X^T X if given.
    lazy=True returns Q as LazyQ(X, R^{-1})."""
    n = X.shape[1]
    if G is None:
        G = gram_dev(X)
    info, Rinv = potrf_inv_dev(G, shift)
    if info:
        return info, None, None
    diag = _diag_host(G, n)
    Q = LazyQ(X, Rinv) if lazy else matmul_dev(X, Rinv, b_upper=True)
    return 0, Q, diag


def orth_speculative_dev(X, lazy_last=False):
    """The CholeskyQR2 route of orth_dev without host synchronisation.

    Every quantity orth_core decides on -- diag(G0) (its trace is ||X||_F^2),
    the two Cholesky infos, diag(R1), diag(R2) -- is left in device buffers;
    returns (Q, probe) where probe is a list of device tensors to read with the
    caller's single synchronisation, and `orth_speculation_holds` replays
    orth_core's decisions on them: True iff orth_core would have taken exactly
    this route (no breakdown, no third pass) and accepted the result, so the
    returned Q is bit-identical to orth_dev's."""
    m, n = X.shape
    diag = device.vector(3 * n)
    infos = torch.zeros(2, dtype=torch.int32, device=X.device)
    work = device.arena().get("potrf_work", int(_native.load().lr_potrf_workspace_doubles(n)))
    G0 = gram_dev(X)
    _native.call("lr_diag_f64", device.ptr(G0), device.ld(G0), n, device.ptr(diag[0:n]), _st())
    R1inv = device.empty(n, n)
    _native.call("lr_potrf_inv_async_f64", n, device.ptr(G0), device.ld(G0), 0.0, device.ptr(R1inv),
                 device.ld(R1inv), device.ptr(work), device.ptr(infos[0:1]), _st())
    _native.call("lr_diag_f64", device.ptr(G0), device.ld(G0), n, device.ptr(diag[n:2 * n]), _st())
    Q1 = matmul_dev(X, R1inv, b_upper=True)
    # ||R1^{-1}||_F^2 for the caller's condition estimate of X
    # (kappa_F(X) = sqrt(trace(G0)) ||R1^{-1}||_F, read with the one sync)
    rstat = _stats_dev_async(R1inv)
    G1 = gram_dev(Q1)
    R2inv = device.empty(n, n)
    _native.call("lr_potrf_inv_async_f64", n, device.ptr(G1), device.ld(G1), 0.0, device.ptr(R2inv),
                 device.ld(R2inv), device.ptr(work), device.ptr(infos[1:2]), _st())
    _native.call("lr_diag_f64", device.ptr(G1), device.ld(G1), n, device.ptr(diag[2 * n:3 * n]), _st())
    Q = LazyQ(Q1, R2inv) if lazy_last else matmul_dev(Q1, R2inv, b_upper=True)
    if isinstance(Q, LazyQ):
        Q.R1inv = R1inv  # Q1 = X R1^{-1}: lets a caller holding Y^T X skip Y^T Q1
    return Q, [diag, infos, rstat]


def _stats_dev_async(X):
    """Device [sum of squares, max |x|, #non-finite] of a block (no sync)."""
    part = device.arena().get("stats_partial_aux", _native.load().lr_stats_partials() + 8)
    out = device.vector(3)
    _native.call("lr_block_stats_f64", device.ptr(X), X.shape[0], X.shape[1], device.ld(X), device.ptr(part),
                 device.ptr(out), _st())
    return out


def orth_speculation_holds(diag_h, infos_h) -> bool:
    """orth_core's decisions on the values orth_speculative_dev recorded."""
    n = diag_h.shape[0] // 3
    if int(infos_h[0]) != 0 or int(infos_h[1]) != 0:
        return False
    tr = float(np.sum(diag_h[0:n]))
    if not (np.isfinite(tr) and tr < 1e300) or tr <= 0.0:
        return False
    scale = float(np.sqrt(tr))
    d1, d2 = diag_h[n:2 * n], diag_h[2 * n:3 * n]
    if not np.all(np.isfinite(d2)) or np.max(np.abs(d2 - 1.0)) > 1e-6:
        return False
    return not np.any(np.abs(d2 * d1) < ORTH_RANK_TOL * scale)


def orth_dev(X, lazy_last=False):
    """Orthonormal basis of range(X) (linalg.py:101-124), device in/out.

    ||X||_F comes from the trace of the first Gram (no extra pass over X);
    a non-finite trace triggers the explicit finiteness check.  lazy_last
    returns the final CholeskyQR pass unformed (LazyQ)."""
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise ValueError(f"orth input must be 2-D with positive dims, got shape {tuple(X.shape)}")
    m, n = X.shape
    if m < n:
        raise ValueError(f"orth requires m >= n, got {m}x{n}")
    return orth_core(X, m, gram_dev, _cholqr_pass, lambda: _fro_from_stats(_check_dev(X, "orth input"), X),
                     lambda G: _diag_host(G, n), lazy_last=lazy_last)


def orth_core(X, m, gram, cholqr, checked_norm, diag, lazy_last=False):
    """CholeskyQR2 / shifted CholeskyQR3 with the reference's collapse test,
    over callables so a row-sharded X (shards.py: gram = local Gram +
    allreduce, m = global rows) runs the same decisions on every rank.
    lazy_last: the last pass of the CholeskyQR2 route comes back as LazyQ
    (cholqr must accept lazy=True); every other route is formed."""
    n = X.shape[1]
    G0 = gram(X)
    tr = float(np.sum(diag(G0)))
    if np.isfinite(tr) and tr < 1e300:
        scale = float(np.sqrt(tr))
    else:
        scale = checked_norm()
    if scale == 0.0:
        raise RankDeficiencyError("cannot orthonormalize a zero matrix")
    info, Q1, d1 = cholqr(X, G=G0)
    if info == 0:
        info2, Q, d2 = cholqr(Q1, lazy=True) if lazy_last else cholqr(Q1)
        if info2 == 0:
            rdiag = d2 * d1
            if np.max(np.abs(d2 - 1.0)) > 1e-6:  # Q1 was far from orthonormal: one more pass
                if isinstance(Q, LazyQ):
                    Q = Q.materialize()
                info3, Q3, d3 = cholqr(Q, lazy=True) if lazy_last else cholqr(Q)
                if info3 == 0:
                    Q, rdiag = Q3, d3 * rdiag
    else:
        info2 = 1
    if info != 0 or info2 != 0:
        # shifted CholeskyQR3 (Fukaya et al.): well defined for any full-rank X
        shift = 11.0 * (m * n + n * (n + 1)) * _U_ROUND * scale * scale
        info, Q1, d1 = cholqr(X, shift)
        if info:
            raise RankDeficiencyError(f"shifted Cholesky failed at column {info - 1}; cannot orthonormalize")
        rdiag = d1
        Q = Q1
        for _ in range(2):
            info, Qn, dn = cholqr(Q)
            if info:
                raise RankDeficiencyError(
                    f"column norm collapse at column {info - 1} (|R[{info - 1},{info - 1}]| = 0.000e+00 < "
                    f"{ORTH_RANK_TOL:.0e} * ||X||_F = {ORTH_RANK_TOL * scale:.3e})")
            Q, rdiag = Qn, dn * rdiag
    rdiag = np.abs(rdiag)
    bad = np.flatnonzero(rdiag < ORTH_RANK_TOL * scale)
    if bad.size:
        j = int(bad[0])
        raise RankDeficiencyError(
            f"column norm collapse at column {j} (|R[{j},{j}]| = {rdiag[j]:.3e} < "
            f"{ORTH_RANK_TOL:.0e} * ||X||_F = {ORTH_RANK_TOL * scale:.3e})")
    return Q


def _public(fn_dev, X, *args):
    is_t = type(X).__module__.startswith("torch")
    out = fn_dev(device.to_device(X), *args)
    return out if is_t else device.to_host(out)


def orth(X):
    """Orthonormal basis of range(X) via CholeskyQR2 on the device."""
    return _public(orth_dev, X)


# -------------------------------------------------------------------- lu_pl

def lu_pl_dev(X, inplace=True):
    """P^T L of partial-pivoting LU (linalg.py:127-150); in place by default."""
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise ValueError(f"lu input must be 2-D with positive dims, got shape {tuple(X.shape)}")
    m, n = X.shape
    if m < n:
        raise ValueError(f"lu_pl requires m >= n, got {m}x{n}")
    if not inplace:
        Y = device.empty(m, n)
        _native.call("lr_copy2d_f64", device.ptr(X), device.ld(X), device.ptr(Y), device.ld(Y), m, n, 0, _st())
        X = Y
    work = device.arena().get("lu_work", int(_native.load().lr_lu_workspace_doubles(m, n)))
    status = (ctypes.c_double * 4)()
    _native.call("lr_lu_pl_f64", m, n, device.ptr(X), device.ld(X), device.ptr(work), status, _st())
    code = status[0]
    if code == -3.0:
        raise ValueError("lu input contains non-finite entries")
    if code == -2.0:
        raise RankDeficiencyError("cannot LU-factor a zero matrix")
    if code >= 0.0:
        j = int(code)
        raise RankDeficiencyError(f"zero pivot at column {j} (|pivot| = {status[1]:.3e} < {status[2]:.3e})")
    return X


def lu_pl(X):
    """Permuted lower-triangular LU factor spanning range(X)."""
    is_t = type(X).__module__.startswith("torch")
    Xd = device.to_device(X)
    out = lu_pl_dev(Xd, inplace=Xd is not X)
    return out if is_t else device.to_host(out)


# ------------------------------------------------------------------ sym_eig

def sym_eig_dev(B, symmetrize=True):
    """(V, d) with d ascending (linalg.py:153-169); B is not modified."""
    n = B.shape[0]
    A = device.empty(n, n)
    if symmetrize:
        _native.call("lr_symmetrize_f64", device.ptr(B), device.ld(B), n, device.ptr(A), device.ld(A), _st())
    else:
        _native.call("lr_copy2d_f64", device.ptr(B), device.ld(B), device.ptr(A), device.ld(A), n, n, 0, _st())
    d = device.vector(n)
    V = device.empty(n, n)
    if EIG_METHOD == "syevd":
        work = device.arena().get("syevd_work", int(_native.load().lr_syevd_workspace_doubles(n)))
        # clusters_host = NULL: the cluster count stays on the device (no stream sync)
        _native.call("lr_syevd_f64", n, device.ptr(A), device.ld(A), device.ptr(d), device.ptr(V), device.ld(V),
                     device.ptr(work), None, _st(), meta={"n": n})
        return V, d
    work = device.arena().get("syevj_work", int(_native.load().lr_syevj_workspace_doubles(n)))
    sweeps = ctypes.c_int(0)
    try:
        _native.call("lr_syevj_f64", n, device.ptr(A), device.ld(A), device.ptr(d), device.ptr(V), device.ld(V),
                     JACOBI_MAX_SWEEPS, device.ptr(work), ctypes.byref(sweeps), _st(), meta={"n": n})
    except NumericalError as exc:
        raise NumericalError(f"symmetric eigensolver did not converge: {_native.last_error()}") from exc
    return V, d


def sym_eig(B):
    """Eigendecomposition of (B + B^T)/2, eigenvalues ascending."""
    Bd = device.to_device(B)
    if Bd.dim() != 2 or Bd.shape[0] < 1 or Bd.shape[1] < 1:
        raise ValueError(f"sym_eig input must be 2-D with positive dims, got shape {tuple(Bd.shape)}")
    _check_dev(Bd, "sym_eig input")
    if Bd.shape[0] != Bd.shape[1]:
        raise ValueError(f"sym_eig needs a square matrix, got {tuple(Bd.shape)}")
    V, d = sym_eig_dev(Bd)
    if type(B).__module__.startswith("torch"):
        return V, d
    return device.to_host(V), device.to_host(d)


# ------------------------------------------------------------------ eig_svd

def gram_spectrum(dh):
    """Singular values sqrt(max(d, 0)) of ascending Gram eigenvalues d, after
    the reference's rank checks (linalg.py:190-198)."""
    n = dh.shape[0]
    dmax = dh[-1]
    if dmax <= 0.0:
        raise RankDeficiencyError("Gram matrix has no positive eigenvalue (zero input?)")
    bad = np.flatnonzero(dh <= GRAM_RANK_TOL * dmax)
    if bad.size:
        raise RankDeficiencyError(
            f"Gram eigenvalue {bad.size} of {n} at/below rank tolerance "
            f"(index {bad[0]}: {dh[bad[0]]:.3e} <= {GRAM_RANK_TOL:.0e} * {dmax:.3e})")
    return np.sqrt(np.maximum(dh, 0.0))


def eig_svd_dev(A, cols=None, check=True, defer=False, G=None):
    """Gram-route SVD of tall A (linalg.py:172-202), device in/out.
    G: A's Gram already formed (the fp32 mode's tensor-core Gram).

    Returns (S_host ascending (all n), V (n x n, sign rule applied),
    U_sel (rows x len(cols)) = A V[:, cols] / S[cols], cols) with cols an
    index array into the ascending order (default: all, ascending).
    """
    if A.dim() != 2 or A.shape[0] < 1 or A.shape[1] < 1:
        raise ValueError(f"eig_svd input must be 2-D with positive dims, got shape {tuple(A.shape)}")
    rows, n = A.shape
    if rows < n:
        raise ValueError(f"eig_svd requires m >= n, got {rows}x{n}")
    if G is None:
        G = gram_dev(A)
    try:
        V, d = sym_eig_dev(G, symmetrize=False)
    except NumericalError:
        _check_dev(A, "oracle_svd input")  # a non-finite input is the reference's ValueError
        raise
    # the lift is queued before the host reads d (see eig_svd_congruent_dev)
    _native.call("lr_fix_signs_f64", device.ptr(V), device.ld(V), n, n, None, 0, 0, _st())
    if cols is None:
        cols = np.arange(n)
    cols = np.asarray(cols, dtype=np.int64)
    Sd = device.vector(n)
    _native.call("lr_gram_spectrum_f64", device.ptr(d), n, device.ptr(Sd), _st())
    B = device.empty(n, cols.shape[0])
    ci = device.int_buffer(cols)
    _native.call("lr_scale_columns_f64", device.ptr(V), device.ld(V), n, device.ptr(ci), cols.shape[0],
                 device.ptr(Sd), 1, device.ptr(B), device.ld(B), _st())
    U = matmul_dev(A, B)

    def finish():
        dh = device.to_host(d)
        # a non-finite input shows as non-finite Gram eigenvalues: only then is
        # the input scanned, for the reference's ValueError (no extra sync before)
        if check and not np.all(np.isfinite(dh)):
            _check_dev(A, "eig_svd input")
        return gram_spectrum(dh)

    finish.reads = [d]  # what finish() will read (device.prefetch_host batches it with the caller's reads)
    if defer:  # the caller queues more work first; finish() reads d and checks the rank
        return finish, V, U, cols
    return finish(), V, U, cols


def eig_svd_congruent_dev(T, Rinv, cols, defer=False, Gt=None):
    """eig_svd_dev of A = T Rinv without forming A (Rinv upper triangular,
    W x W): Gram(A) = Rinv^T Gram(T) Rinv (two W^3 products instead of an
    n x W x W one), U_sel = T (Rinv V[:, cols] / S[cols]).  Same returns as
    eig_svd_dev.  Gt: Gram(T) already formed."""
    rows, n = T.shape
    if Gt is None:
        Gt = gram_dev(T)
    H = matmul_dev(Gt, Rinv, b_upper=True)   # Gram(T) Rinv
    G = matmul_tn_dev(Rinv, H)               # Rinv^T Gram(T) Rinv
    try:
        V, d = sym_eig_dev(G, symmetrize=True)   # (G + G^T)/2, as sym_eig does
    except NumericalError:
        _check_dev(T, "eig_svd input")
        raise
    # the lift is queued before the host reads d: the rank checks run while
    # the GPU lifts (a rank error discards the lift and raises as before)
    _native.call("lr_fix_signs_f64", device.ptr(V), device.ld(V), n, n, None, 0, 0, _st())
    cols = np.asarray(cols, dtype=np.int64)
    Sd = device.vector(n)
    _native.call("lr_gram_spectrum_f64", device.ptr(d), n, device.ptr(Sd), _st())
    B = device.empty(n, cols.shape[0])
    ci = device.int_buffer(cols)
    _native.call("lr_scale_columns_f64", device.ptr(V), device.ld(V), n, device.ptr(ci), cols.shape[0],
                 device.ptr(Sd), 1, device.ptr(B), device.ld(B), _st())
    U = matmul_dev(T, tri_mul_dev(Rinv, B))

    def finish():
        dh = device.to_host(d)
        if not np.all(np.isfinite(dh)):  # non-finite input: the reference's ValueError
            _check_dev(T, "eig_svd input")
        return gram_spectrum(dh)

    finish.reads = [d]
    if defer:
        return finish, V, U, cols
    return finish(), V, U, cols


def tri_mul_dev(Rinv, B):
    """Rinv (upper triangular, W x W) @ B (W x c), dense small product."""
    return matmul_dev(Rinv, B)


def eig_svd(A) -> SvdResult:
    """Economic SVD of a tall full-column-rank matrix via its Gram matrix;
    singular values ascending."""
    Ad = device.to_device(A)
    S, V, U, _ = eig_svd_dev(Ad)
    if type(A).__module__.startswith("torch"):
        return SvdResult(U, device.f64_buffer(S), V, "ascending")
    return SvdResult(device.to_host(U), S, device.to_host(V), "ascending")


# --------------------------------------------------------------- oracle_svd

JACOBI_MAX_SWEEPS = 30     # sweeps rotating every pair (the reference's tc_rq fallbacks need > 12)
JACOBI_NOISE_SWEEPS = 30   # further sweeps with noise-against-noise pairs skipped
# columns of the dense SVD with S <= DENSE_NULL_FLOOR * S[0] get an orthonormal
# completion instead of B / S (1e-300: exact zeros only)
DENSE_NULL_FLOOR = float(__import__("os").environ.get("LR_DENSE_NULL_FLOOR", "1e-300"))


def _tall_dense_svd_dev(A):
    """Descending SVD of tall A (rows >= n) on the device, to dgesdd's
    absolute accuracy (linalg.py:205-221): the Gram route (syrk + syevd)
    gives V0 whose B = A V0 has nearly orthogonal columns; one-sided Jacobi
    sweeps (lr_jacobi_sweep_f64, rotations accumulated into V) orthogonalise
    B's columns to sqrt(rows) eps, S = their norms (error ~ eps s_max even for
    null directions, where the Gram route alone stops at ~sqrt(eps) s_max),
    U = B / S, null directions completed from a seeded Gaussian block and
    re-orthonormalised by CholeskyQR2 (good columns barely move)."""
    rows, n = A.shape
    st = _st()
    G = gram_dev(A)
    try:
        V0, _d = sym_eig_dev(G, symmetrize=False)
    except NumericalError:
        _check_dev(A, "oracle_svd input")  # a non-finite input is the reference's ValueError
        raise
    Vd = device.empty(n, n)  # eigenvectors, descending
    oi = device.int_buffer(np.arange(n - 1, -1, -1))
    _native.call("lr_scale_columns_f64", device.ptr(V0), device.ld(V0), n, device.ptr(oi), n, None, 0,
                 device.ptr(Vd), device.ld(Vd), st)
    # the preconditioner must be orthogonal to working precision: inverse
    # iteration leaves eigenvectors of small-gap eigenvalue pairs only
    # eps / gap orthogonal (~1e-8 at a 1e-8 gap); two CholeskyQR passes on the
    # n x n block fix that (the rotations below preserve orthogonality)
    for _ in range(2):
        info, Qv, _dv = _cholqr_pass(Vd)
        if info:
            break
        Vd = Qv
    B = matmul_dev(A, Vd)
    Bt = device.empty(n, rows)
    _native.call("lr_transpose_f64", device.ptr(B), device.ld(B), rows, n, device.ptr(Bt), device.ld(Bt), st)
    Vt = device.empty(n, n)
    _native.call("lr_transpose_f64", device.ptr(Vd), device.ld(Vd), n, n, device.ptr(Vt), device.ld(Vt), st)
    off = device.vector(1)
    norms = device.vector(n)
    tol = float(np.sqrt(rows)) * 2.0 * _U_ROUND
    noise2 = 0.0
    skipped = False
    for sweep in range(JACOBI_MAX_SWEEPS + JACOBI_NOISE_SWEEPS):
        if sweep == JACOBI_MAX_SWEEPS:
            # not converged: the pairs still rotating are noise against noise
            # (exactly dependent columns of a tall A); stop rotating those
            _native.call("lr_row_norms_f64", device.ptr(Bt), device.ld(Bt), n, rows, device.ptr(norms), st)
            noise = float(np.max(device.to_host(norms))) * max(rows, n) * 2.0 * _U_ROUND
            noise2, skipped = noise * noise, True
        _native.call("lr_jacobi_sweep_f64", n, rows, device.ptr(Bt), device.ld(Bt), device.ptr(Vt), device.ld(Vt),
                     tol, noise2, device.ptr(off), st)
        if float(device.to_host(off)[0]) == 0.0:
            break
    else:
        raise NumericalError("dense SVD: one-sided Jacobi did not converge")
    _native.call("lr_row_norms_f64", device.ptr(Bt), device.ld(Bt), n, rows, device.ptr(norms), st)
    Sj = device.to_host(norms)
    perm = np.argsort(-Sj, kind="stable")
    S = Sj[perm]
    # U = B / S for every column with a nonzero norm: Jacobi leaves the
    # columns orthogonal RELATIVE to their norms, so even noise-level ones
    # normalise to orthonormal vectors inside span(A) -- as dgesdd's U lies in
    # span(Q) of A's QR -- and only exactly-zero columns need a completion
    # noise-level columns left unrotated among themselves are not orthogonal:
    # complete them like exact zeros
    floor = S[0] * (max(rows, n) * 2.0 * _U_ROUND if skipped else DENSE_NULL_FLOOR) if S[0] > 0 else np.inf
    good = S > floor
    # U = B[:, perm] / S (good columns), V = Vt^T[:, perm]
    _native.call("lr_transpose_f64", device.ptr(Bt), device.ld(Bt), n, rows, device.ptr(B), device.ld(B), st)
    pi = device.int_buffer(perm)
    Ssafe = device.f64_buffer(np.where(Sj > floor, Sj, 1.0))  # floor: S[0] * DENSE_NULL_FLOOR
    U = device.empty(rows, n)
    _native.call("lr_scale_columns_f64", device.ptr(B), device.ld(B), rows, device.ptr(pi), n, device.ptr(Ssafe), 1,
                 device.ptr(U), device.ld(U), st)
    _native.call("lr_transpose_f64", device.ptr(Vt), device.ld(Vt), n, n, device.ptr(Vd), device.ld(Vd), st)
    V = device.empty(n, n)
    _native.call("lr_scale_columns_f64", device.ptr(Vd), device.ld(Vd), n, device.ptr(pi), n, None, 0,
                 device.ptr(V), device.ld(V), st)
    nbad = int((~good).sum())
    if nbad:
        from .rng import gaussian_matrix_device

        Z = gaussian_matrix_device(0x5EED, rows, nbad)
        _native.call("lr_copy2d_f64", device.ptr(Z), device.ld(Z), device.ptr(U[:, n - nbad:]), device.ld(U),
                     rows, nbad, 0, st)
        # re-orthonormalise (columns keep their order; good columns barely move)
        for _ in range(2):
            info, Qn, _dd = _cholqr_pass(U)
            if info:
                shift = 11.0 * (rows * n + n * (n + 1)) * _U_ROUND * float(n)
                info, Qn, _dd = _cholqr_pass(U, shift)
                if info:
                    raise NumericalError("dense SVD: could not orthonormalize the left factor")
            U = Qn
    _native.call("lr_fix_signs_f64", device.ptr(V), device.ld(V), n, n, device.ptr(U), device.ld(U), rows, st)
    return U, S, V


def oracle_svd_dev(A):
    """Full economic SVD, descending (linalg.py:205-221) -> (U, S_host, V)."""
    _check_dev(A, "oracle_svd input")
    m, n = A.shape
    if min(m, n) > ORACLE_SVD_CAP:
        raise SizeCapError(f"oracle SVD capped at min(m,n) <= {ORACLE_SVD_CAP}, got {m}x{n}")
    if m >= n:
        return _tall_dense_svd_dev(A)
    At = device.empty(n, m)
    _native.call("lr_transpose_f64", device.ptr(A), device.ld(A), m, n, device.ptr(At), device.ld(At), _st())
    U2, S, V2 = _tall_dense_svd_dev(At)  # A^T = U2 S V2^T  ->  A = V2 S U2^T
    # sign rule on A's V (= U2): first nonzero of each column >= 0
    _native.call("lr_fix_signs_f64", device.ptr(U2), device.ld(U2), n, m, device.ptr(V2), device.ld(V2), m, _st())
    return V2, S, U2


def oracle_svd(A) -> SvdResult:
    """Dense economic SVD (descending) on the device; desk-scale only."""
    U, S, V = oracle_svd_dev(device.to_device(A))
    return SvdResult(device.to_host(U), S, device.to_host(V), "descending")
