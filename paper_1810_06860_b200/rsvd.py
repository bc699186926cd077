"""Randomized truncated SVDs of sparse matrices, on the device.

Drop-in for /root/reference/pkg/src/lowrank/rsvd.py:
  rsvd_bki  Alg. 5: LU-normalised Krylov blocks H_0..H_p written straight
            into column slices of one m x W device block (no hstack), QR of
            the block, B^T = Y^T Q on the CSC copy, Gram-route SVD with only
            the top-k window lifted                          (rsvd.py:200-231)
  rsvd_pi   Alg. 4: LU power iteration, Gram-route final basis (rsvd.py:168-197)
  rsvd_basic Alg. 1 comparator (QR each product, dense small SVD)
                                                              (rsvd.py:134-165)
  qb_error  ||A - U S V^T||_F / ||A||_F without densifying   (rsvd.py:234-254)
Rank deficiency reroutes through the dense device SVD when allow_fallback,
else re-raises with the same advice suffixes (rsvd.py:81-126).

Omega is gaussian_matrix(RngState(seed), n, k+s).  `omega="host"` (the
default, OMEGA_SOURCE) draws it with numpy on the host -- the reference's own
arithmetic, bit for bit, split over a thread pool (rng.normals_column_major)
-- and uploads it in draw order for a device-side transpose; the SVT loop
prefetches the next fresh call's draw while the GPU works.  `omega="device"`
generates it on the GPU from the same numpy Philox stream (uniform words
bit-exact, normals within 4e-15 of the host values --
tests/test_gpu_kernels.py::test_device_gaussian_matches_host), so no n x w
block crosses PCIe.  The parity suite runs both.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, device
from .errors import RankDeficiencyError
from .linalg import (DevSvd, LazyQ, SvdResult, eig_svd_congruent_dev, eig_svd_dev, gram_tf32x3_dev, lu_pl_dev, matmul_dev,
                     oracle_svd_dev, orth_dev, orth_speculation_holds, orth_speculative_dev)
from .rng import RngState, gaussian_matrix, gaussian_matrix_device
from .sparse import SparseMatrix, frobenius, spmm_dev, spmm_dev32, spmm_t_dev, spmm_t_dev32

# Omega's producer: "host" (the parity default: numpy's own draw, north_star's
# "the same Gaussian test matrix passed in from the host") or "device"
# (lr_gaussian_f64, the same Philox words, normals within 4e-15; no PCIe)
OMEGA_SOURCE = "host"
# rsvd_bki leaves the last CholeskyQR pass unformed (linalg.LazyQ): Y^T Q and
# Q V run through Q1 and R2^{-1}; Subspace.Q forms Q only when asked.
LAZY_LAST_PASS = True
LAZY_MIN_FLOPS = 1 << 30  # m * W^2 below this: form Q (the GEMM is a few microseconds)
# rsvd_bki checks LU statuses and orth's decisions with one read after the
# basis is built, redoing the call on the careful path when one is unusual
SPECULATIVE = True
# Y^T Q1 for the unformed basis Q1 = H R1^{-1}: (Y^T H) R1^{-1}, where Y^T H's
# blocks are the Krylov products Y^T H_i already computed (plus Y^T H_p) -- one
# narrow product and an n x W x W GEMM instead of the W-wide one.  Rounding in
# Y^T H is amplified by kappa(H) <= kappa_F(H) = sqrt(trace(G0)) ||R1^{-1}||_F
# (both on the device already); used only while kappa_F(H) <= KRYLOV_REUSE_KAPPA,
# i.e. at most ~2e-10 relative error in Y^T Q1 (the parity bar is 1e-8).
KRYLOV_REUSE = True
KRYLOV_REUSE_KAPPA = 1e6  # cfg4 job: kappa_F(H) 2e3 .. 1.2e5 (profiles/r02u_cfg4_timeline.txt)
REUSE_STATS = {"used": 0, "kappa_gate": 0, "kappas": [], "skipped": 0}
# (m, n, nnz, w, p) -> the last call of that shape tripped the kappa gate: the
# next one does not queue the reuse projection at all (cfg2 at p = 5 trips it
# every call: a dropped projection is an n x W x W product, a W x W eigensolve
# and two lifts, ~7 ms of a 23 ms call).  kappa_F(H) is still read on every
# call, so the route comes back as soon as one call passes the gate.
_REUSE_GATED = {}


@dataclass
class RsvdParams:
    """k target rank, p power/Krylov parameter, s oversampling, seed."""

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

    def check_against(self, A: SparseMatrix, krylov: bool = False) -> None:
        width = (self.k + self.s) * ((self.p + 1) if krylov else 1)
        limit = min(A.rows, A.cols)
        if width > limit:
            raise ValueError(f"sketch width {width} exceeds min(m, n) = {limit}; reduce k, s or p")


class Subspace:
    """Orthonormal sketch basis (device resident; `.Q` downloads lazily)."""

    def __init__(self, Q, provenance: str, p: int, fallbacks: int = 0):
        self._Q = Q
        self.provenance = provenance
        self.p = p
        self.fallbacks = fallbacks
        self._Qh = None

    @property
    def Q(self) -> np.ndarray:
        if isinstance(self._Q, np.ndarray):
            return self._Q
        if self._Qh is None:
            self._Qh = device.to_host(self.Q_dev)
        return self._Qh

    @property
    def Q_dev(self):
        if isinstance(self._Q, np.ndarray):
            self._Q = device.to_device(self._Q)
        if isinstance(self._Q, LazyQ) or hasattr(self._Q, "materialize"):
            self._Q = self._Q.materialize()  # an unformed product, or a deferred gather (shards._GatheredQ)
        return self._Q

    @property
    def Q_any(self):
        """The device basis as stored: a tensor or an unformed LazyQ."""
        if isinstance(self._Q, np.ndarray):
            self._Q = device.to_device(self._Q)
        return self._Q

    @property
    def width(self) -> int:
        return int(self._Q.shape[1])


class _Fallback:
    __slots__ = ("enabled", "count", "advice")

    def __init__(self, enabled: bool, advice: str):
        self.enabled, self.count, self.advice = enabled, 0, advice

    def fail(self, exc):
        if not self.enabled:
            if self.advice is None:
                raise exc
            raise RankDeficiencyError(f"{exc}; {self.advice}") from exc
        self.count += 1


def _copy(src, dst):
    _native.call("lr_copy2d_f64", device.ptr(src), device.ld(src), device.ptr(dst), device.ld(dst),
                 src.shape[0], src.shape[1], 0, device.stream())


def _omega(seed: int, n: int, w: int, source: str):
    if source == "device":
        return gaussian_matrix_device(seed, n, w)
    return omega_from_host(seed, n, w)


def _overlap_draw_with_upload(A: SparseMatrix, seed: int, n: int, w: int, source: str) -> None:
    """A call on a matrix whose device mirror is not built yet (the public API
    from host arrays): start the host draw of Omega in the background, then
    upload the pattern / values and build the transpose index meanwhile."""
    if source != "host" or A._pattern is not None:
        return
    from .rng import prefetch_normals

    prefetch_normals(seed, n, w)
    A.pattern()
    A.device_values()


OMEGA_STATS = {"assembled_on_device": 0, "prefetched_upload": 0, "host_draw": 0}
_OMEGA_VERIFY = __import__("os").environ.get("LR_OMEGA_VERIFY") == "1"


def omega_from_host(seed: int, n: int, w: int):
    """Omega = gaussian_matrix(RngState(seed), n, w) drawn on the HOST with
    numpy's own arithmetic (bit-identical to the reference's draw; threaded,
    rng.normals_column_major) into page-locked memory in draw (column-major)
    order, uploaded, and transposed into the row-major device block on the
    GPU (lr_transpose_f64) -- the host never does the strided transpose."""
    import torch

    from .rng import superset_on_device, take_normals, take_normals_device

    device.require_cuda()
    count = n * w
    pre = take_normals_device(seed, n, w)
    sup = superset_on_device(seed, n, w) if (pre is None and count) else None
    OMEGA_STATS["assembled_on_device" if sup is not None else ("prefetched_upload" if pre is not None
                                                                else "host_draw")] += 1
    if sup is not None:
        # the Box-Muller halves of a range of widths are on the GPU already:
        # this width's Omega is one multiply per entry there (bit-identical
        # to the host draw), written row-major directly
        R, cs, ready = sup.dev
        cur = torch.cuda.current_stream()
        cur.wait_event(ready)
        # the buffers live in the upload stream's pool: when a staging slot outgrows them they are
        # freed while this stream may still have the kernel below queued
        R.record_stream(cur)
        cs.record_stream(cur)
        if not sup.counted:
            sup.counted = True
            device.TRAFFIC["h2d"] += 8 * (int(R.numel()) + int(cs.numel()))
        Om = device.empty(n, w)
        _native.call("lr_omega_assemble_f64", device.ptr(R), device.ptr(cs), (count + 1) // 2 - sup.p_lo, n, w,
                     device.ptr(Om), device.ld(Om), device.stream())
        sup.mark_consumed(cur)  # the staging slot's device copies are rewritten only after this kernel
        if _OMEGA_VERIFY:  # diagnostic: the assembled block against the reference draw, bit for bit
            from .rng import gaussian_matrix

            ref = gaussian_matrix(RngState(seed), n, w)
            got = device.to_host(Om)
            if not np.array_equal(got, ref):
                bad = np.argwhere(got != ref)
                raise AssertionError(f"device-assembled Omega(seed={seed}, {n}x{w}) differs from the host draw at "
                                     f"{bad.shape[0]} entries, first {bad[0].tolist()}, last {bad[-1].tolist()}; "
                                     f"superset widths [{sup.w_lo}, {sup.w_hi}], slot gen {sup._slot.gen} vs {sup._gen}")
        return Om
    if pre is not None:  # the prefetch thread already copied it (upload stream)
        dv, ready = pre
        cur = torch.cuda.current_stream()
        cur.wait_event(ready)
        dv.record_stream(cur)
        Zt = dv[:max(count, 1)].view(w, n) if count else device.empty(w, n)
    else:
        host = take_normals(seed, n, w)
        Zt = device.vector(count).view(w, n) if count else device.empty(w, n)
        Zt.view(-1).copy_(host[:count], non_blocking=True)
    device.TRAFFIC["h2d"] += 8 * count
    Om = device.empty(n, w)
    _native.call("lr_transpose_f64", device.ptr(Zt), n, w, n, device.ptr(Om), device.ld(Om), device.stream())
    return Om


def _lu_block(block, fb: _Fallback):
    """LU-normalise a device block in place; dense-SVD basis on fallback."""
    keep = None
    if fb.enabled:
        keep = device.empty(*block.shape)
        _copy(block, keep)
    try:
        lu_pl_dev(block)
    except RankDeficiencyError as exc:
        fb.fail(exc)
        U, _, _ = oracle_svd_dev(keep)
        _copy(U, block)


def _lu_block_async(block, status):
    """LU-normalise a device block in place, its status left on the device."""
    m, n = block.shape
    work = device.arena().get("lu_work", int(_native.load().lr_lu_workspace_doubles(m, n)))
    _native.call("lr_lu_pl_async_f64", m, n, device.ptr(block), device.ld(block), device.ptr(work),
                 device.ptr(status), device.stream())


def _orthonormalize(X, fb: _Fallback, lazy_last=False):
    try:
        return orth_dev(X, lazy_last=lazy_last)
    except RankDeficiencyError as exc:
        fb.fail(exc)
        return oracle_svd_dev(X)[0]


def _windowed_small_svd(Bt, idx, fb: _Fallback, Rinv=None, defer=False, G=None):
    """eig_svd of Bt (n x W) keeping the ascending-order columns idx (given in
    the output order).  Returns (S_sel host, V_small[:, idx] device,
    U_small[:, idx] device).  Falls back to the dense SVD (ascending).
    With Rinv the matrix is Bt @ Rinv, never formed unless the fallback
    needs it.  defer: returns (finish, Vsel, Usel) with the work queued and
    finish() -> (S_sel, Vsel, Usel) reading the eigenvalues (the rank check
    and the fallback happen there)."""
    try:
        if Rinv is None:
            fin, V, U, cols = eig_svd_dev(Bt, cols=idx, defer=True, G=G)
        else:
            fin, V, U, cols = eig_svd_congruent_dev(Bt, Rinv, idx, defer=True, Gt=G)
        Vsel = device.empty(V.shape[0], len(idx))
        ci = device.int_buffer(cols)
        _native.call("lr_scale_columns_f64", device.ptr(V), device.ld(V), V.shape[0], device.ptr(ci), len(idx),
                     None, 0, device.ptr(Vsel), device.ld(Vsel), device.stream())
    except RankDeficiencyError as exc:
        out = _windowed_fallback(Bt, idx, fb, Rinv, exc)
        return (lambda: out, out[1], out[2]) if defer else out

    def finish():
        try:
            return fin()[cols], Vsel, U
        except RankDeficiencyError as exc:
            return _windowed_fallback(Bt, idx, fb, Rinv, exc)

    finish.reads = getattr(fin, "reads", [])
    return (finish, Vsel, U) if defer else finish()


def _windowed_fallback(Bt, idx, fb: _Fallback, Rinv, exc):
    """_windowed_small_svd's dense-SVD route after a rank failure."""
    fb.fail(exc)
    if Rinv is not None:
        Bt = matmul_dev(Bt, Rinv, b_upper=True)
    Ud, Sd, Vd = oracle_svd_dev(Bt)  # descending
    W = Bt.shape[1]
    desc = W - 1 - np.asarray(idx)  # ascending index -> descending position
    ci = device.int_buffer(desc)
    Vsel = device.empty(Vd.shape[0], len(idx))
    Usel = device.empty(Ud.shape[0], len(idx))
    _native.call("lr_scale_columns_f64", device.ptr(Vd), device.ld(Vd), Vd.shape[0], device.ptr(ci), len(idx),
                 None, 0, device.ptr(Vsel), device.ld(Vsel), device.stream())
    _native.call("lr_scale_columns_f64", device.ptr(Ud), device.ld(Ud), Ud.shape[0], device.ptr(ci), len(idx),
                 None, 0, device.ptr(Usel), device.ld(Usel), device.stream())
    return Sd[desc], Vsel, Usel


# fp32 mode: the eigSVD Gram of the fp32 product on the tcgen05 tensor cores
# (3xTF32); False: the fp64 DMMA Gram of the widened product
GRAM_TF32 = __import__("os").environ.get("LR_GRAM_TF32", "1") != "0"


def _spmm_t_prec(Y: SparseMatrix, X, precision: str, with_gram: bool = False):
    """Y^T X in the requested precision; the fp32 product comes back fp64.
    with_gram: returns (product, its Gram or None) -- the fp32 product's Gram
    formed from the fp32 values on the tensor cores (GRAM_TF32)."""
    if precision == "fp32" and int(X.shape[1]) >= 2:
        T32 = spmm_t_dev32(Y, device.to_f32(X))
        T = device.to_f64(T32)
        if with_gram:
            return T, (gram_tf32x3_dev(T32) if GRAM_TF32 else None)
        return T
    T = spmm_t_dev(Y, X)
    return (T, None) if with_gram else T


def project_and_solve(Y: SparseMatrix, Q, k: int, fb: _Fallback, precision: str = "fp64",
                      download: bool = False, T_pre=None, defer=False):
    """B^T = Y^T Q, small SVD, lift: the shared tail of Alg. 5 steps 8-10,
    recycle_q and rsvd_pi.  Returns the top-k DevSvd (descending).
    download: V's device->host copy starts (side stream) before U is lifted.
    defer: everything is queued and a callable returned; calling it reads the
    eigenvalues (rank check, dense fallback if needed) and gives the DevSvd."""
    W = int(Q.shape[1])
    idx = np.arange(W - 1, W - k - 1, -1)  # top-k of the ascending order, descending
    lazy = isinstance(Q, LazyQ)
    G = None
    if lazy:
        # Q = Q1 Rinv unformed: B^T = (Y^T Q1) Rinv, U = Q1 (Rinv V_small)
        T, G = (T_pre, None) if T_pre is not None else _spmm_t_prec(Y, Q.base, precision, with_gram=True)
        fin, Vsel, Usel = _windowed_small_svd(T, idx, fb, Rinv=Q.Rinv, defer=True, G=G)
    else:
        Bt, G = (T_pre, None) if T_pre is not None else _spmm_t_prec(Y, Q, precision, with_gram=True)
        fin, Vsel, Usel = _windowed_small_svd(Bt, idx, fb, defer=True, G=G)

    def lift(Vs, Us):
        pend = device.to_host_async(Us) if download else None
        U = matmul_dev(Q.base, matmul_dev(Q.Rinv, Vs)) if lazy else matmul_dev(Q, Vs)
        return U, pend

    U, pend = lift(Vsel, Usel)

    def finish():
        S_sel, Vs, Us = fin()
        U2, pend2 = (U, pend) if Vs is Vsel else lift(Vs, Us)  # the fallback replaced the small factors
        return DevSvd(U2, device.f64_buffer(S_sel), Us, np.asarray(S_sel, dtype=np.float64), pend2)

    finish.reads = getattr(fin, "reads", [])
    return finish if defer else finish()


class Prestart:
    """The first product of an inner SVD queued ahead of its call (the SVT
    loop queues it behind the fused step, before reading the residual):
    kind "bki": H (m x w (p_max + 1), block 0 = LU(Y Omega)) and the LU status
    vector; kind "recycle-q": T = Y^T Q of the cached basis."""

    def __init__(self, kind, **kw):
        self.kind = kind
        self.__dict__.update(kw)

    def matches(self, params: "RsvdParams") -> bool:
        return (self.kind == "bki" and params.k == self.k and params.s == self.s and params.seed == self.seed
                and params.p <= self.p_max)


def bki_prestart(A: SparseMatrix, k: int, s: int, seed: int, p_max: int, precision: str = "fp64"):
    """Alg. 5 steps 1-2 of a coming rsvd_bki call: Omega (seed), H_0 = A Omega
    and its LU (status left on the device), into an H block wide enough for
    p_max Krylov steps.  None when the call will not use it (fp32 mode, the
    careful path)."""
    if not SPECULATIVE or _check_precision(precision) == "fp32":
        return None
    w = k + s
    m, n = A.shape
    Om = _omega(seed, n, w, OMEGA_SOURCE)
    H = device.empty(m, w * (p_max + 1))
    lu_status = device.vector(4 * (p_max + 1))
    spmm_dev(A, Om, out=H[:, 0:w])
    _lu_block_async(H[:, 0:w], lu_status[0:3])
    return Prestart("bki", k=k, s=s, seed=seed, p_max=p_max, H=H, lu_status=lu_status)


def recycle_prestart(Y: SparseMatrix, cached: "Subspace", precision: str = "fp64"):
    """The product B^T = Y^T Q (Q1 for an unformed basis) of a coming recycle_q."""
    Q = cached.Q_any
    base = Q.base if isinstance(Q, LazyQ) else Q
    return Prestart("recycle-q", Q=Q, T=_spmm_t_prec(Y, base, precision))


def _check_precision(precision: str) -> str:
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
    return precision


def _krylov_orth(A: SparseMatrix, Om, params: RsvdParams, spec: bool, fp32: bool, lazy: bool, fb: _Fallback,
                 pre: Prestart = None, keep_T: bool = False):
    """Alg. 5 steps 1-7 from a given Omega: Krylov blocks H_0..H_p (LU-
    normalised) and the basis.  spec: LU statuses and the CholeskyQR route's
    decisions stay on the device (no host synchronisation at all: the body
    can be captured in a CUDA graph).  Returns (H, Q, lu_status, probe)."""
    w = params.k + params.s
    W = w * (params.p + 1)
    m, n = A.shape
    if pre is not None:  # H_0 and its LU already queued (bki_prestart)
        H = pre.H[:, :W]
        lu_status = pre.lu_status[:4 * (params.p + 1)]
    else:
        lu_status = device.vector(4 * (params.p + 1)) if spec else None
        H = device.empty(m, W)

    def normalise(i):
        if spec:
            _lu_block_async(H[:, i * w:(i + 1) * w], lu_status[4 * i:4 * i + 3])
        else:
            _lu_block(H[:, i * w:(i + 1) * w], fb)

    if fp32:
        H32, T32 = device.empty32(m, w), device.empty32(n, w)
        spmm_dev32(A, device.to_f32(Om), out=H32)
        device.to_f64(H32, out=H[:, 0:w])
    elif pre is None:
        spmm_dev(A, Om, out=H[:, 0:w])
    if pre is None:
        normalise(0)
    keep_T = keep_T and not fp32
    T_all = device.empty(n, W) if keep_T else None  # Y^T H, block by block
    T = None if fp32 else device.empty(n, w)
    for i in range(1, params.p + 1):
        if fp32:
            device.to_f32(H[:, (i - 1) * w:i * w], out=H32)
            spmm_t_dev32(A, H32, out=T32)
            spmm_dev32(A, T32, out=H32)
            device.to_f64(H32, out=H[:, i * w:(i + 1) * w])
        else:
            if keep_T:
                T = T_all[:, (i - 1) * w:i * w]
            spmm_t_dev(A, H[:, (i - 1) * w:i * w], out=T)
            spmm_dev(A, T, out=H[:, i * w:(i + 1) * w])
        normalise(i)
    if keep_T:
        spmm_t_dev(A, H[:, params.p * w:W], out=T_all[:, params.p * w:W])
    if spec:
        Q, probe = orth_speculative_dev(H, lazy_last=lazy)
    else:
        Q, probe = _orthonormalize(H, fb, lazy_last=lazy), None
    if keep_T and isinstance(Q, LazyQ):
        Q.T_all = T_all
    return H, Q, lu_status, probe


def rsvd_bki_dev(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False, omega=None,
                 precision: str = "fp64", download: bool = False, _speculate: bool = True, pre: Prestart = None):
    """Device Alg. 5 -> (DevSvd, Q device, fallbacks).

    precision="fp32" (north_star's optional fp32 mode, singular values within
    1e-4): the sparse products run on fp32 values and fp32 blocks (half the
    gathered bytes); LU, CholeskyQR, the eigensolver and the lifts stay fp64
    on the converted blocks."""
    params.check_against(A, krylov=True)
    fp32 = _check_precision(precision) == "fp32" and params.k + params.s >= 2
    fb = _Fallback(allow_fallback, "Krylov blocks are near-collinear, reduce p or use a larger matrix")
    w = params.k + params.s
    W = w * (params.p + 1)
    m, n = A.shape
    # small blocks (launch-bound, e.g. cfg1's 1000 x 64): forming Q is cheaper
    # than the extra small products of the unformed route
    lazy = LAZY_LAST_PASS and m * W * W >= LAZY_MIN_FLOPS
    # Speculation: the LU statuses and orth's decisions stay on the device and
    # are read with ONE synchronisation after the basis is built; if any of
    # them is not the common case (a zero pivot, a Cholesky breakdown, a third
    # CholeskyQR pass, a rank collapse) the call is redone on the careful path,
    # which makes every decision as it goes -- so results, errors and
    # fallbacks are exactly the careful path's.  (The speculative steps have
    # no host synchronisation and were captured as a CUDA graph once: -9 %
    # per steady-state cfg1-sized call, but ~6 ms per capture, and the SVT
    # loop's k changes make captures outnumber replays -- not kept.)
    spec = SPECULATIVE and _speculate
    use_pre = (pre is not None and spec and not fp32 and (omega or OMEGA_SOURCE) == OMEGA_SOURCE
               and pre.matches(params))
    if not use_pre:
        _overlap_draw_with_upload(A, params.seed, n, w, omega or OMEGA_SOURCE)
    Om = None if use_pre else _omega(params.seed, n, w, omega or OMEGA_SOURCE)
    reuse_ok = KRYLOV_REUSE and spec and lazy and not fp32 and params.p >= 1
    gate_key = (m, n, int(A.nnz), w, params.p)
    reuse = reuse_ok and not _REUSE_GATED.get(gate_key, False)
    if reuse_ok and not reuse:
        REUSE_STATS["skipped"] += 1
    H, Q, lu_status, probe = _krylov_orth(A, Om, params, spec, fp32, lazy, fb, pre=pre if use_pre else None,
                                          keep_T=reuse)
    T_pre = None
    fin_spec = None
    if spec and reuse and isinstance(Q, LazyQ) and getattr(Q, "T_all", None) is not None:
        # queue the projection on the reused Krylov products before the one
        # host read of this call (LU statuses, orth decisions, kappa): it
        # stands when all of them hold (the common case), else it is dropped
        fin_spec = project_and_solve(A, Q, params.k, fb, "fp64", download=download,
                                     T_pre=matmul_dev(Q.T_all, Q.R1inv, b_upper=True), defer=True)
    if spec:
        # one batched device -> host transfer for everything this call reads (LU statuses, orth's
        # decisions, ||R1^{-1}||, the small eigenvalues): one wait, then plain host arrays
        device.prefetch_host([lu_status, probe[0], probe[1], probe[2]] + list(getattr(fin_spec, "reads", [])))
        try:
            st = device.to_host(lu_status).reshape(-1, 4)[:, :3]
            diag_h, infos_h = device.to_host(probe[0]), device.to_host(probe[1])
            if not np.all(st[:, 0] == -1.0):  # an LU decision differed: redo the whole call
                return rsvd_bki_dev(A, params, allow_fallback, omega, precision, download, _speculate=False)
            if not orth_speculation_holds(diag_h, infos_h):
                # the Krylov blocks are exactly the careful path's (H is untouched
                # by the speculative orth): only the orthonormalisation is redone
                Q = _orthonormalize(H, fb, lazy_last=lazy)
            elif reuse_ok and isinstance(Q, LazyQ):
                Wn = diag_h.shape[0] // 3
                kappa = float(np.sqrt(np.sum(diag_h[0:Wn]) * device.to_host(probe[2])[0]))
                if len(REUSE_STATS["kappas"]) < 4096:
                    REUSE_STATS["kappas"].append(kappa)
                passes = bool(np.isfinite(kappa) and kappa <= KRYLOV_REUSE_KAPPA)
                if len(_REUSE_GATED) > 4096:
                    _REUSE_GATED.clear()
                _REUSE_GATED[gate_key] = not passes
                if fin_spec is not None and passes:
                    REUSE_STATS["used"] += 1
                    res = fin_spec()  # the speculatively queued projection stands
                    if isinstance(Q, LazyQ):
                        Q.T_all = Q.R1inv = None  # the cached basis (reuse-q) must not pin them
                    return res, Q, fb.count
                if fin_spec is not None:
                    REUSE_STATS["kappa_gate"] += 1  # queued and dropped
            if isinstance(Q, LazyQ):
                Q.T_all = Q.R1inv = None
        finally:
            device.clear_prefetched()  # nothing prefetched outlives the tensors it mirrors
    res = project_and_solve(A, Q, params.k, fb, "fp32" if fp32 else "fp64", download=download, T_pre=T_pre)
    return res, Q, fb.count


def rsvd_bki(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False, *, omega=None,
             precision: str = "fp64"):
    """Rank-k randomized SVD by block Krylov iteration (descending).
    precision="fp32": the optional fp32 mode (sparse products in fp32)."""
    res, Q, nfb = rsvd_bki_dev(A, params, allow_fallback, omega, precision, download=True)
    return res.to_host(), Subspace(Q, "bki", params.p, nfb)


def rsvd_pi_dev(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False, omega=None):
    params.check_against(A)
    fb = _Fallback(allow_fallback, "increase s or reduce k")
    w = params.k + params.s
    m, n = A.shape
    _overlap_draw_with_upload(A, params.seed, n, w, omega or OMEGA_SOURCE)
    Om = _omega(params.seed, n, w, omega or OMEGA_SOURCE)
    Q = spmm_dev(A, Om)
    T = device.empty(n, w)
    for _ in range(params.p):
        _lu_block(Q, fb)
        spmm_t_dev(A, Q, out=T)
        spmm_dev(A, T, out=Q)
    # final basis through the Gram-route SVD (all w columns, ascending)
    try:
        _, _, Q, _ = eig_svd_dev(Q)
    except RankDeficiencyError as exc:
        fb.fail(exc)
        Q = oracle_svd_dev(Q)[0]
    Bt = spmm_t_dev(A, Q)
    idx = np.arange(params.k + params.s - 1, params.s - 1, -1)  # window [s, k+s), descending
    S_sel, Vsel, Usel = _windowed_small_svd(Bt, idx, fb)
    U = matmul_dev(Q, Vsel)
    return DevSvd(U, device.f64_buffer(S_sel), Usel, np.asarray(S_sel)), Q, fb.count


def rsvd_pi(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False, *, omega=None):
    """Rank-k randomized SVD with LU-renormalised power iteration."""
    res, Q, nfb = rsvd_pi_dev(A, params, allow_fallback, omega)
    return res.to_host(), Subspace(Q, "pi", params.p, nfb)


def rsvd_basic(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False, *, omega=None):
    """Alg. 1 comparator: orthonormalise after every product, dense SVD of
    the projected matrix (rsvd.py:134-165)."""
    params.check_against(A)
    fb = _Fallback(allow_fallback, "matrix rank is likely below k+s, reduce k")
    w = params.k + params.s
    Om = _omega(params.seed, A.cols, w, omega or OMEGA_SOURCE)
    Q = _orthonormalize(spmm_dev(A, Om), fb)
    for _ in range(params.p):
        G = _orthonormalize(spmm_t_dev(A, Q), fb)
        Q = _orthonormalize(spmm_dev(A, G), fb)
    Bt = spmm_t_dev(A, Q)  # (Q^T A)^T, n x w; SVD of B = Q^T A from that of B^T
    Ub, S, Vb = oracle_svd_dev(Bt)  # B^T = Ub S Vb^T -> B = Vb S Ub^T
    _native.call("lr_fix_signs_f64", device.ptr(Ub), device.ld(Ub), Ub.shape[0], Ub.shape[1], device.ptr(Vb),
                 device.ld(Vb), Vb.shape[0], device.stream())
    k = params.k
    U = matmul_dev(Q, Vb)
    res = SvdResult(device.to_host(U)[:, :k], S[:k].copy(), device.to_host(Ub)[:, :k], "descending")
    return res, Subspace(Q, "pi", params.p, fb.count)


def qb_error(A: SparseMatrix, res: SvdResult) -> float:
    """||A - U S V^T||_F / ||A||_F via ||A||^2 - 2<A V S, U> + ||S||^2."""
    U, S, V = res.U, res.S, res.V
    if U.shape[0] != A.rows or V.shape[0] != A.cols:
        raise ValueError(f"factor dims {U.shape[0]}x{V.shape[0]} do not match matrix {A.shape}")
    if U.shape[1] != S.shape[0] or V.shape[1] != S.shape[0]:
        raise ValueError("factor rank mismatch")
    a_norm = frobenius(A.data)
    if a_norm == 0.0:
        raise ValueError("relative error undefined for a zero matrix")
    k = int(S.shape[0])
    if k == 0:
        return 1.0
    Sh = np.asarray(S, dtype=np.float64)
    Vd = device.to_device(V)
    P = spmm_dev(A, Vd)  # m x k
    Ud = device.to_device(U)
    # cross = sum_ij P_ij S_j U_ij : scale U's columns by S, then a Frobenius inner product
    Sd = device.f64_buffer(Sh)
    US = device.empty(U.shape[0], k)
    _native.call("lr_scale_columns_f64", device.ptr(Ud), device.ld(Ud), U.shape[0], None, k, device.ptr(Sd), 0,
                 device.ptr(US), device.ld(US), device.stream())
    # <P, US> = trace(P^T US): sum of the diagonal of a k x k product
    G = device.empty(k, k)
    from .linalg import matmul_tn_dev

    matmul_tn_dev(P, US, out=G)
    d = device.vector(k)
    _native.call("lr_diag_f64", device.ptr(G), device.ld(G), k, device.ptr(d), device.stream())
    cross = float(np.sum(device.to_host(d)))
    sq = a_norm * a_norm - 2.0 * cross + float(Sh @ Sh)
    return float(np.sqrt(max(sq, 0.0))) / a_norm
