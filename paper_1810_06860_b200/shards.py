"""Sharded SVT / rSVD-BKI: one matrix spread over ranks.

One process per GPU.  The observed pattern is cut twice, by nnz-balanced
prefix sums (ShardPlan):
  row shard  R_g  CSR block Y[R_g, :]   -> products Y X      (rows R_g)
  col shard  C_g  CSR block Y[:, C_g]   -> products Y^T X    (rows C_g, via
                                            the block's CSC copy)
Every m x . dense block is either replicated (Krylov blocks H_i, the basis
Q) or row-sharded by R_g (U factors); every n x . block is replicated
(T, Omega) or row-sharded by C_g (V factors).  Per fresh BKI call:

  Omega (n x w)            generated on every rank from the same Philox seed
  H_0 = Y Omega            local rows -> allgather -> GEPP replicated
  T = Y^T H_{i-1}          local rows -> allgather; H_i = Y T -> allgather -> GEPP
  Q = orth(H)              CholeskyQR2 on row shards: local Gram -> allreduce
                           -> replicated Cholesky -> local Q rows -> allgather
  B^T = Y^T Q              local rows (C_g); eig_svd: local Gram -> allreduce
                           -> replicated eigensolver -> V rows C_g, U = Q V rows R_g
  SVT step                 CSR side needs full V (allgather n x r), CSC side full
                           U (allgather m x r); both sides compute each entry
                           with the same kernel from the same U row / V row, so
                           the two value copies of Y stay bit-identical; the
                           residual partials are allgathered and summed in rank
                           order on every rank.

Allreduce results are identical on every rank, so every replicated solve and
every host decision (ranks, escalation, fallbacks, convergence) agrees across
ranks without further communication.  The single-GPU engine
(completion.DeviceEngine) is the world-size-1 special case of the same loop;
results at N ranks equal it within fp64 rounding (Gram sums are split
differently), never bit-for-bit.

The collectives go through torch.distributed (`Exchange`): NCCL between GPUs,
gloo for the host-side tests (tests/test_shards_gloo.py runs world size 2 on
the CPU with a numpy kernel set injected through `kernels=`).  The product
kernel set is DeviceKernels -- the sm_100a library; nothing here computes on
the host.
"""

from __future__ import annotations

import numpy as np

from . import _native, device
from .errors import DataError, RankDeficiencyError
from .linalg import DevSvd, SvdResult, gram_spectrum, orth_core
from .rsvd import RsvdParams, Subspace, _Fallback
from .sparse import ObservationSet, SparseMatrix

__all__ = ["ShardPlan", "Exchange", "DeviceKernels", "ShardedEngine", "svt_sharded", "rsvd_bki_sharded"]


# ------------------------------------------------------------------ plan

def balanced_bounds(ptr, parts: int) -> np.ndarray:
    """Contiguous cut of len(ptr)-1 rows into `parts` blocks with about
    nnz/parts entries each (prefix-sum search); every block gets >= 1 row."""
    ptr = np.asarray(ptr, dtype=np.int64)
    size = ptr.shape[0] - 1
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    if size < parts:
        raise ValueError(f"cannot cut {size} rows into {parts} non-empty shards")
    nnz = int(ptr[-1])
    b = np.empty(parts + 1, dtype=np.int64)
    b[0], b[parts] = 0, size
    for g in range(1, parts):
        target = (g * nnz) // parts
        i = int(np.searchsorted(ptr, target, side="left"))
        b[g] = min(max(i, b[g - 1] + 1), size - (parts - g))
    return b


class ShardPlan:
    """Row bounds (CSR indptr) and column bounds (CSC indptr) of a pattern."""

    def __init__(self, indptr, t_indptr, world: int):
        self.world = int(world)
        self.row_bounds = balanced_bounds(indptr, world)
        self.col_bounds = balanced_bounds(t_indptr, world)
        ip, tp = np.asarray(indptr), np.asarray(t_indptr)
        self.row_nnz = ip[self.row_bounds[1:]] - ip[self.row_bounds[:-1]]
        self.col_nnz = tp[self.col_bounds[1:]] - tp[self.col_bounds[:-1]]

    def rows(self, g: int):
        return int(self.row_bounds[g]), int(self.row_bounds[g + 1])

    def cols(self, g: int):
        return int(self.col_bounds[g]), int(self.col_bounds[g + 1])

    def describe(self) -> dict:
        return {"row_bounds": self.row_bounds.tolist(), "col_bounds": self.col_bounds.tolist(),
                "row_nnz": self.row_nnz.tolist(), "col_nnz": self.col_nnz.tolist()}


# ------------------------------------------------------------ collectives

class Exchange:
    """The sharded path's collectives over torch.distributed: uneven row
    allgather, in-place sum allreduce, small scalar allgather.  Counts bytes
    moved for the bench line."""

    def __init__(self, group=None, always_collective=False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, "none"
        # world size 1 short-circuits to local copies unless asked to run the
        # collectives anyway (the one-GPU NCCL test exercises them that way)
        self.collective = self.world > 1 or (always_collective and self.backend != "none")
        self.bytes = 0
        self.calls = 0

    def gather_rows(self, local, bounds, out):
        """out[bounds[g]:bounds[g+1]] = rank g's `local`, on every rank."""
        import torch

        w = int(local.shape[1])
        if not self.collective:
            if out.data_ptr() != local.data_ptr() or out.stride() != local.stride():
                out.copy_(local)
            return out
        if w == 0:
            return out
        counts = np.diff(bounds)
        cmax = int(counts.max())
        send = torch.empty((cmax, w), dtype=local.dtype, device=local.device)
        send[: local.shape[0]].copy_(local)
        if local.shape[0] < cmax:
            send[local.shape[0]:].zero_()
        recv = torch.empty((self.world * cmax, w), dtype=local.dtype, device=local.device)
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            self.dist.all_gather(list(recv.chunk(self.world)), send, group=self.group)
        for g in range(self.world):
            c = int(counts[g])
            out[int(bounds[g]):int(bounds[g]) + c].copy_(recv[g * cmax:g * cmax + c])
        self.bytes += int(recv.numel()) * 8
        self.calls += 1
        return out

    def allreduce_sum(self, t):
        if not self.collective:
            return t
        flat = t if t.is_contiguous() else t.contiguous()
        self.dist.all_reduce(flat, group=self.group)
        if flat is not t:
            t.copy_(flat)
        self.bytes += int(flat.numel()) * 8
        self.calls += 1
        return t

    def gather_scalars(self, vec) -> np.ndarray:
        """(world, k) host array of every rank's k-vector (a tensor on the
        engine's device), identical on all ranks."""
        import torch

        if not self.collective:
            return vec.detach().cpu().numpy().reshape(1, -1).astype(np.float64)
        k = int(vec.numel())
        send = vec.reshape(-1).contiguous()
        recv = torch.empty((self.world * k,), dtype=send.dtype, device=send.device)
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            self.dist.all_gather(list(recv.chunk(self.world)), send, group=self.group)
        self.calls += 1
        return recv.cpu().numpy().reshape(self.world, k).astype(np.float64)


# ------------------------------------------------------------ kernel set

class DeviceKernels:
    """Per-rank operations of the sharded engine on the sm_100a library
    (the same entry points the single-GPU path calls)."""

    def __init__(self):
        _native.load()

    # memory
    def empty(self, rows, cols):
        return device.empty(rows, cols)

    def vector(self, values):
        return device.f64_buffer(np.asarray(values, dtype=np.float64))

    def from_host(self, a):
        return device.to_device(np.ascontiguousarray(a, dtype=np.float64))

    def to_host(self, t):
        return device.to_host(t)

    def copy(self, src, dst):
        if src.shape[0] * src.shape[1]:
            _native.call("lr_copy2d_f64", device.ptr(src), device.ld(src), device.ptr(dst), device.ld(dst),
                         src.shape[0], src.shape[1], 0, device.stream())

    # sparse blocks
    def block(self, rows, cols, indptr, indices, data, prep=None, slot=0):
        """Device block; prep[slot] caches its host prep (transpose index,
        schedules) across re-uploads of the same pattern."""
        A = SparseMatrix(rows, cols, indptr, indices, data)
        if prep is not None and prep[slot] is not None:
            A._hprep = prep[slot]
        A.device_values()
        if prep is not None:
            prep[slot] = A._hprep
        return A

    def scaled_block(self, A, scale):
        """scale * A's values on A's pattern, formed on the device."""
        return A.scaled_on_device(scale)

    def block_like(self, A, data):
        B = SparseMatrix(A.rows, A.cols, A.indptr, A.indices, data)
        B.share_pattern(A)
        B.device_values()
        return B

    def host_values(self, A):
        return A.data

    def values(self, A):
        return A.device_values()[0]

    def densify(self, A):
        return A.densify()

    def spmm(self, A, X, out):
        from .sparse import spmm_dev

        return spmm_dev(A, X, out=out)

    def spmm_t(self, A, X, out):
        from .sparse import spmm_t_dev

        return spmm_t_dev(A, X, out=out)

    def svt_step(self, A, m_vals, U, S_dev, V, r, step):
        """Fused residual + update of A's two value copies; device [sumsq, max|x-m|]."""
        dp = A.pattern()
        npart = int(_native.load().lr_svt_step_partials())
        part = device.arena().get("svt_partial", npart + 8)
        out2 = device.vector(2)
        yc = A.device_values_csr()
        _native.call("lr_svt_step_f64", device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), dp.csr.rows,
                     device.ptr(dp.csr.items), dp.csr.n_items, device.ptr(U), device.ld(U) if r else 1,
                     device.ptr(S_dev), device.ptr(V), device.ld(V) if r else 1, r, device.ptr(m_vals),
                     device.ptr(yc), None, device.ptr(dp.inv_perm), float(step), 1,
                     device.ptr(part), npart, device.ptr(out2), device.stream(),
                     meta={"nnz": A.nnz, "m": A.rows, "n": A.cols, "r": r, "csc_scatter": False})
        A._host_stale = True
        A._dvals32 = None
        A.mark_csc_stale()
        return out2

    def project(self, A, U, S_dev, V, r):
        from .sparse import project_pattern_dev

        return project_pattern_dev(U, S_dev, V, A) if r else device.vector(A.nnz).zero_()

    def stats(self, x):
        """Device [sum of squares, max|x|, #non-finite] of a vector / block."""
        if x.dim() == 1:
            rows, cols, ldx = x.shape[0], 1, 1
        else:
            rows, cols, ldx = x.shape[0], x.shape[1], device.ld(x)
        out = device.vector(3)
        if rows * cols == 0:
            return out.zero_()
        part = device.arena().get("stats_partial", _native.load().lr_stats_partials() + 8)
        _native.call("lr_block_stats_f64", device.ptr(x), rows, cols, ldx, device.ptr(part), device.ptr(out),
                     device.stream())
        return out

    def scaled_stats(self, x, big):
        xs = x.reshape(-1, 1) if x.dim() == 1 else x
        rows, cols = xs.shape
        y = device.empty(rows, cols)
        scale = device.f64_buffer(np.full(max(cols, 1), big))
        _native.call("lr_scale_columns_f64", device.ptr(xs), device.ld(xs) if x.dim() == 2 else 1, rows, None,
                     cols, device.ptr(scale), 1, device.ptr(y), device.ld(y), device.stream())
        return self.stats(y)

    def power(self, x0_host):
        from .sparse import PowerIteration

        return PowerIteration(x0_host)

    # dense
    def gram(self, X):
        from .linalg import gram_dev

        return gram_dev(X)

    def matmul(self, A, B, b_upper=False):
        from .linalg import matmul_dev

        return matmul_dev(A, B, b_upper=b_upper)

    def potrf_inv(self, G, shift=0.0):
        from .linalg import potrf_inv_dev

        return potrf_inv_dev(G, shift)

    def diag(self, G):
        from .linalg import _diag_host

        return _diag_host(G, G.shape[0])

    def sym_eig(self, G):
        from .linalg import sym_eig_dev

        V, d = sym_eig_dev(G, symmetrize=False)
        return V, device.to_host(d)

    def fix_signs(self, V):
        n = V.shape[0]
        _native.call("lr_fix_signs_f64", device.ptr(V), device.ld(V), n, V.shape[1], None, 0, 0, device.stream())

    def select_columns(self, V, cols, S=None):
        """V[:, cols] (divided column-wise by S[cols] when S is given)."""
        cols = np.asarray(cols, dtype=np.int64)
        B = device.empty(V.shape[0], cols.shape[0])
        ci = device.int_buffer(cols)
        Sd = device.f64_buffer(S) if S is not None else None
        _native.call("lr_scale_columns_f64", device.ptr(V), device.ld(V), V.shape[0], device.ptr(ci),
                     cols.shape[0], device.ptr(Sd), 1 if S is not None else 0, device.ptr(B), device.ld(B),
                     device.stream())
        return B

    def lu_pl_async(self, X, status):
        """LU-normalise X in place with its status left on the device
        (status[0] == -1: pivots as usual; anything else: the caller replays
        the careful path)."""
        m, n = X.shape
        work = device.arena().get("lu_work", int(_native.load().lr_lu_workspace_doubles(m, n)))
        _native.call("lr_lu_pl_async_f64", m, n, device.ptr(X), device.ld(X), device.ptr(work), device.ptr(status),
                     device.stream())

    def lu_pl(self, X):
        from .linalg import lu_pl_dev

        return lu_pl_dev(X)

    def gaussian(self, seed, rows, cols):
        """Omega(seed) on this rank: the parity default draws on the host
        (every rank the same bits; the SVT loop prefetches it as on one GPU),
        omega="device" generates it on the GPU."""
        from . import rsvd as _rsvd
        from .rng import gaussian_matrix_device

        if _rsvd.OMEGA_SOURCE == "host":
            return _rsvd.omega_from_host(seed, rows, cols)
        return gaussian_matrix_device(seed, rows, cols)

    def dense_svd(self, X):
        from .linalg import oracle_svd_dev

        return oracle_svd_dev(X)


# ---------------------------------------------------------------- engine

class ShardedEngine:
    """completion._svt_loop's matrix side spread over ranks; also the
    sharded rSVD-BKI (`bki`).  Factors U are row-sharded by R_g, V by C_g."""

    @property
    def omega_source(self):  # the single-GPU default: every rank draws the same host Omega (prefetched)
        from . import rsvd as _rsvd

        return _rsvd.OMEGA_SOURCE

    def __init__(self, obs: ObservationSet, exchange: Exchange = None, kernels=None):
        self.ex = exchange if exchange is not None else Exchange()
        self.K = kernels if kernels is not None else DeviceKernels()
        self.rank, self.world = self.ex.rank, self.ex.world
        if isinstance(self.K, DeviceKernels):
            # every rank builds the train CSR on its own device (the same
            # validation and bit-exact ordering as the single-GPU engine; the
            # host lexsort of cfg4's 18M cells costs seconds) and cuts its two
            # blocks out of it there
            phi = obs.train_matrix()
            if phi.nnz == 0:
                raise DataError("no observed entries to complete from")
            if phi._dev_csr is not None:
                self._setup_device(phi)
                return
        else:
            r, c, v = obs.subset(ObservationSet.TRAIN)
            phi = SparseMatrix.from_coo(obs.m, obs.n, r, c, v)  # host: same ordering / validation everywhere
            if phi.nnz == 0:
                raise DataError("no observed entries to complete from")
        self._setup(phi)

    @classmethod
    def from_matrix(cls, A: SparseMatrix, exchange: Exchange = None, kernels=None) -> "ShardedEngine":
        self = cls.__new__(cls)
        self.ex = exchange if exchange is not None else Exchange()
        self.K = kernels if kernels is not None else DeviceKernels()
        self.rank, self.world = self.ex.rank, self.ex.world
        self._setup(A, A.__dict__.setdefault("_shard_cache", {}))
        return self

    def _setup(self, phi: SparseMatrix, cache: dict = None) -> None:
        """Cut phi into this rank's row and column blocks.  The integer side
        (plan, slices, block patterns and their host prep) is cached in
        `cache` (A._shard_cache for from_matrix), like the single-GPU host
        prep, so a re-upload re-slices only the values."""
        K = self.K
        self.m, self.n = phi.shape
        self.nnz = phi.nnz
        key = (self.world, self.rank)
        st = cache.get(key) if cache is not None else None
        if st is None:
            t_indptr = np.zeros(self.n + 1, dtype=np.int64)  # CSC offsets only (no host argsort)
            np.cumsum(np.bincount(phi.indices, minlength=self.n), out=t_indptr[1:])
            plan = ShardPlan(phi.indptr, t_indptr, self.world)
            r0, r1 = plan.rows(self.rank)
            c0, c1 = plan.cols(self.rank)
            ip, ix = phi.indptr, phi.indices
            lo, hi = int(ip[r0]), int(ip[r1])
            sel = np.flatnonzero((ix >= c0) & (ix < c1))
            cptr = np.zeros(self.m + 1, dtype=np.int64)
            np.cumsum(np.bincount(phi.coo_rows()[sel], minlength=self.m), out=cptr[1:])
            st = {"plan": plan, "lo": lo, "hi": hi, "rptr": ip[r0:r1 + 1] - lo, "ridx": ix[lo:hi], "sel": sel,
                  "cptr": cptr, "cidx": ix[sel] - c0, "prep": [None, None]}
            if cache is not None:
                cache[key] = st
        self.plan = st["plan"]
        self.r0, self.r1 = self.plan.rows(self.rank)
        self.c0, self.c1 = self.plan.cols(self.rank)
        dv = phi.data
        self.phi_r = K.block(self.r1 - self.r0, self.n, st["rptr"], st["ridx"], dv[st["lo"]:st["hi"]],
                             prep=st["prep"], slot=0)
        self.phi_c = K.block(self.m, self.c1 - self.c0, st["cptr"], st["cidx"], dv[st["sel"]],
                             prep=st["prep"], slot=1)
        self.m_r = K.values(self.phi_r)
        self.m_c = K.values(self.phi_c)
        self.Y_r, self.Y_c = self.phi_r, self.phi_c  # rsvd on the observed matrix itself until start()
        self.m_norm = None

    def _setup_device(self, phi: SparseMatrix) -> None:
        """_setup for a device-built CSR (ObservationSet.train_matrix): the
        plan from the host offsets and the device column counts, the row block
        as a slice of the CSR arrays, the column block by one masked selection
        in CSR order (the entries a host `flatnonzero` would pick, in the same
        order).  A rank that holds the whole matrix keeps one block."""
        import torch

        K = self.K
        self.m, self.n = phi.shape
        self.nnz = phi.nnz
        ptr_d, idx_d, vals_d = phi._dev_csr
        if vals_d is None:
            vals_d = phi.device_values()[0]
        ip = phi.indptr
        counts = torch.bincount(idx_d.long(), minlength=self.n)
        t_indptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(counts.cpu().numpy(), out=t_indptr[1:])
        self.plan = plan = ShardPlan(ip, t_indptr, self.world)
        self.r0, self.r1 = r0, r1 = plan.rows(self.rank)
        self.c0, self.c1 = c0, c1 = plan.cols(self.rank)
        if (r0, r1, c0, c1) == (0, self.m, 0, self.n):
            self.phi_r = self.phi_c = phi
        else:
            lo, hi = int(ip[r0]), int(ip[r1])
            # fresh allocations: every array of a block starts on an allocation boundary
            self.phi_r = SparseMatrix.from_device_csr(
                r1 - r0, self.n, ip[r0:r1 + 1] - lo, (ptr_d[r0:r1 + 1] - lo).contiguous(), idx_d[lo:hi].clone(),
                vals_d[lo:hi].clone())
            sel = torch.nonzero((idx_d >= c0) & (idx_d < c1)).view(-1)  # CSR order
            row_of = torch.searchsorted(ptr_d[1:].long().contiguous(), sel, right=True)
            ccount = torch.bincount(row_of, minlength=self.m)
            cptr_h = np.zeros(self.m + 1, dtype=np.int64)
            np.cumsum(ccount.cpu().numpy(), out=cptr_h[1:])
            self.phi_c = SparseMatrix.from_device_csr(
                self.m, c1 - c0, cptr_h, torch.from_numpy(cptr_h.astype(np.int32)).to(idx_d.device),
                (idx_d[sel] - c0).to(torch.int32), vals_d[sel].contiguous())
            del sel, row_of, ccount
        self.phi_r.device_values()
        if self.phi_c is not self.phi_r:
            self.phi_c.device_values()
        self.m_r = K.values(self.phi_r)
        self.m_c = K.values(self.phi_c)
        self.Y_r, self.Y_c = self.phi_r, self.phi_c
        self.m_norm = None

    # ------------------------------------------------------------ helpers
    def vector(self, values):
        return self.K.vector(values)

    def gather_m(self, local, out=None):
        if out is None:
            out = self.K.empty(self.m, local.shape[1])
        return self.ex.gather_rows(local, self.plan.row_bounds, out)

    def gather_n(self, local, out=None):
        if out is None:
            out = self.K.empty(self.n, local.shape[1])
        return self.ex.gather_rows(local, self.plan.col_bounds, out)

    def _reduced_gram(self, X):
        G = self.K.gram(X)
        return self.ex.allreduce_sum(G)

    def _global_stats(self, x) -> np.ndarray:
        return self.ex.gather_scalars(self.K.stats(x))  # (world, 3)

    def _global_norm(self, x) -> float:
        st = self._global_stats(x)
        sumsq, big = float(np.sum(st[:, 0])), float(np.max(st[:, 1]))
        if big == 0.0:
            return 0.0
        if np.isfinite(sumsq) and 1e-150 < big < 1e150:
            return float(np.sqrt(sumsq))
        st2 = self.ex.gather_scalars(self.K.scaled_stats(x, big))
        return float(big * np.sqrt(np.sum(st2[:, 0])))

    def _check_finite(self, X, name):
        if np.sum(self._global_stats(X)[:, 2]):
            raise ValueError(f"{name} contains non-finite entries")

    # --------------------------------------------------- loop interface
    def observed_norm(self) -> float:
        return self._global_norm(self.m_r)

    def spectral_norm(self, rng) -> float:
        from .sparse import _SPECTRAL_BATCH, _SPECTRAL_MAX_ITERS

        K = self.K
        pw = K.power(rng.normal_pairs(self.n))
        # unit-stride columns: the power-update kernel reads z as a flat vector
        y_loc = K.vector(np.zeros(self.r1 - self.r0)).view(-1, 1)
        y = K.vector(np.zeros(self.m)).view(-1, 1)
        z_loc = K.vector(np.zeros(self.c1 - self.c0)).view(-1, 1)
        z = K.vector(np.zeros(self.n)).view(-1, 1)
        for it in range(_SPECTRAL_MAX_ITERS):
            if it and it % _SPECTRAL_BATCH == 0 and pw.done():
                break
            K.spmm(self.phi_r, pw.x, out=y_loc)
            self.gather_m(y_loc, out=y)
            K.spmm_t(self.phi_c, y, out=z_loc)
            self.gather_n(z_loc, out=z)
            pw.update(z)
        return pw.result()

    @property
    def _one_block(self) -> bool:
        """This rank's row block and column block are the same entries (one
        rank holds the whole matrix): one copy of Y serves both sides."""
        return (self.r0, self.r1, self.c0, self.c1) == (0, self.m, 0, self.n)

    def start(self, scale: float) -> None:
        """Y = scale * P_Phi(M) on both blocks, formed on the device from the
        resident value copies (completion.py:335; as DeviceEngine.start)."""
        K = self.K
        self.Y_r = K.scaled_block(self.phi_r, scale)
        self.Y_c = self.Y_r if self._one_block else K.scaled_block(self.phi_c, scale)

    def step(self, U_s, S_s, V_s, r: int, step: float):
        return self.step_launch(U_s, S_s, V_s, r, step)(), None

    def step_launch(self, U_s, S_s, V_s, r: int, step: float):
        """The fused step of both blocks queued on the stream; returns a
        callable that gathers the ranks' partial sums and returns the
        residual (DeviceEngine.step_launch: the SVT loop queues the next inner
        SVD's first product behind the step before it waits for the residual)."""
        K = self.K
        S_dev = K.vector(S_s) if r else K.vector(np.zeros(0))
        if r:
            V_full = self.gather_n(V_s)
            U_full = self.gather_m(U_s)
        else:
            V_full, U_full = V_s, U_s
        # the row block's CSR copy serves Y X, the column block's CSC copy Y^T X:
        # each step updates its block's CSR values (the column block's CSC copy
        # is refreshed on demand by one gather, as on one GPU); a rank holding
        # the whole matrix steps its one copy once
        part = K.svt_step(self.Y_r, self.m_r, U_s, S_dev, V_full, r, step)
        if self.Y_c is not self.Y_r:
            K.svt_step(self.Y_c, self.m_c, U_full, S_dev, V_s, r, step)

        def finish():
            st = self.ex.gather_scalars(part)
            sumsq, big = float(np.sum(st[:, 0])), float(np.max(st[:, 1]))
            if big == 0.0:
                return 0.0
            if np.isfinite(sumsq) and 1e-150 < big < 1e150:
                return float(np.sqrt(sumsq)) / self.m_norm
            # partial sums out of range: the scaled norm of x - m, x recomputed from the factors
            x = K.project(self.Y_r, U_s, S_dev, V_full, r)
            return self._global_norm(x - self.m_r) / self.m_norm

        return finish

    def prestart(self, plan):
        """Queue the first product of the next iteration's fresh BKI call
        behind the fused step (DeviceEngine.prestart): Omega, H_0 = Y Omega
        (local rows, allgather) and its LU with the status left on the device.
        None for a recycle or on a kernel set without the asynchronous LU."""
        from . import rsvd as _rsvd

        K = self.K
        if plan[0] != "bki" or not (_rsvd.SPECULATIVE and hasattr(K, "lu_pl_async")):
            return None
        _, k, s, seed, p_max = plan
        w = k + s
        Om = K.gaussian(seed, self.n, w)
        H = K.empty(self.m, w * (p_max + 1))
        status = K.vector(np.zeros(4 * (p_max + 1)))
        H_loc = K.empty(self.r1 - self.r0, w)
        K.spmm(self.Y_r, Om, out=H_loc)
        self.gather_m(H_loc, out=H[:, 0:w])
        K.lu_pl_async(H[:, 0:w], status[0:3])
        return _rsvd.Prestart("bki", k=k, s=s, seed=seed, p_max=p_max, H=H, lu_status=status)

    def factors_host(self, U_s, V_s, r: int):
        if not r:
            return np.zeros((self.m, 0)), np.zeros((self.n, 0))
        return self.K.to_host(self.gather_m(U_s)), self.K.to_host(self.gather_n(V_s))

    # ------------------------------------------------------ inner SVDs
    def _empty(self, k=0):
        K = self.K
        return DevSvd(K.empty(self.r1 - self.r0, k), K.vector(np.zeros(k)), K.empty(self.c1 - self.c0, k),
                      np.zeros(k))

    def _lu_block(self, block, fb: _Fallback):
        K = self.K
        keep = None
        if fb.enabled:
            keep = K.empty(*block.shape)
            K.copy(block, keep)
        try:
            K.lu_pl(block)
        except RankDeficiencyError as exc:
            fb.fail(exc)
            U, _, _ = K.dense_svd(keep)
            K.copy(U, block)

    def _cholqr(self, X, shift=0.0, G=None):
        K = self.K
        if G is None:
            G = self._reduced_gram(X)
        info, Rinv = K.potrf_inv(G, shift)
        if info:
            return info, None, None
        Q = K.matmul(X, Rinv, b_upper=True)
        if self._passes is not None:
            self._passes.append((X, Q, Rinv, shift, G))  # the pass chain, for the Krylov reuse in bki
        return 0, Q, K.diag(G)

    _passes = None  # a list while bki orthonormalises its Krylov block

    def _chain(self, X, Q):
        """The Rinv factors of the CholeskyQR passes that turned X into Q
        (Q = X R_1^{-1} R_2^{-1} ...), and whether the first was unshifted;
        None when Q is not such a chain of X."""
        by_out = {id(q): (x, r, sh, g) for x, q, r, sh, g in self._passes}
        chain, cur, first = [], Q, None
        while id(cur) in by_out:
            x, r, sh, g = by_out[id(cur)]
            chain.append(r)
            first = (sh, g)
            cur = x
        if cur is not X or not chain:
            return None
        return chain[::-1], first

    def _orth_rows(self, X_loc):
        """orth of the row-sharded block whose local rows are X_loc."""
        return orth_core(X_loc, self.m, self._reduced_gram, self._cholqr,
                         lambda: (self._check_finite(X_loc, "orth input"), self._global_norm(X_loc))[1],
                         self.K.diag)

    def _eig_svd(self, A_loc, cols):
        """eig_svd of the row-sharded n x W block whose local rows are A_loc
        (rows C_g): returns (S ascending, V replicated, U_loc, cols)."""
        K = self.K
        G = self._reduced_gram(A_loc)
        if not np.isfinite(np.sum(K.diag(G))):
            self._check_finite(A_loc, "eig_svd input")
        V, d = K.sym_eig(G)
        S = gram_spectrum(d)
        K.fix_signs(V)
        cols = np.asarray(cols, dtype=np.int64)
        B = K.select_columns(V, cols, S)
        return S, V, K.matmul(A_loc, B), cols

    def _windowed(self, Bt_loc, idx, fb: _Fallback):
        K = self.K
        try:
            S, V, U_loc, cols = self._eig_svd(Bt_loc, idx)
            return S[cols], K.select_columns(V, cols), U_loc
        except RankDeficiencyError as exc:
            fb.fail(exc)
            Bt = self.gather_n(Bt_loc)
            Ud, Sd, Vd = K.dense_svd(Bt)  # descending
            W = Bt.shape[1]
            desc = W - 1 - np.asarray(idx)
            return Sd[desc], K.select_columns(Vd, desc), K.select_columns(Ud, desc)[self.c0:self.c1]

    def _project_and_solve(self, Q, k: int, fb: _Fallback, Bt_loc=None, Q_loc=None) -> DevSvd:
        """Bt_loc / Q_loc given (the Krylov reuse): Y^T Q's rows C_g and Q's
        rows R_g, the full Q never needed."""
        K = self.K
        W = int(Q.shape[1]) if Q is not None else int(Q_loc.shape[1])
        if Bt_loc is None:
            Bt_loc = K.spmm_t(self.Y_c, Q, out=K.empty(self.c1 - self.c0, W))
        idx = np.arange(W - 1, W - k - 1, -1)
        S_sel, Vsel, Usel = self._windowed(Bt_loc, idx, fb)
        U_loc = K.matmul(Q_loc if Q_loc is not None else Q[self.r0:self.r1], Vsel)
        S_sel = np.asarray(S_sel, dtype=np.float64)
        return DevSvd(U_loc, K.vector(S_sel), Usel, S_sel)

    def bki(self, rp: RsvdParams, allow_fallback: bool = True, _speculate: bool = True, pre=None):
        """Sharded Alg. 5 -> (DevSvd with local factor rows, Q replicated, fallbacks).
        Like the single-GPU route, the Krylov blocks' LU statuses stay on the
        device and are read once after the loop; an unusual one replays the
        call on the careful path (every rank reads the same replicated
        statuses, so the ranks agree)."""
        from . import rsvd as _rsvd

        K = self.K
        rp.check_against(self, krylov=True)
        fb = _Fallback(allow_fallback, "Krylov blocks are near-collinear, reduce p or use a larger matrix")
        spec = _speculate and _rsvd.SPECULATIVE and hasattr(K, "lu_pl_async")
        w = rp.k + rp.s
        W = w * (rp.p + 1)
        mg, ng = self.r1 - self.r0, self.c1 - self.c0
        use_pre = pre is not None and spec and pre.kind == "bki" and pre.matches(rp)
        status = None
        if spec:
            status = pre.lu_status[:4 * (rp.p + 1)] if use_pre else K.vector(np.zeros(4 * (rp.p + 1)))

        def normalise(i):
            if spec:
                K.lu_pl_async(H[:, i * w:(i + 1) * w], status[4 * i:4 * i + 3])
            else:
                self._lu_block(H[:, i * w:(i + 1) * w], fb)

        H_loc = K.empty(mg, w)
        if use_pre:  # H_0 and its LU were queued behind the last fused step (prestart)
            H = pre.H[:, :W]
        else:
            Om = K.gaussian(rp.seed, self.n, w)
            H = K.empty(self.m, W)
            K.spmm(self.Y_r, Om, out=H_loc)
            self.gather_m(H_loc, out=H[:, 0:w])
            normalise(0)
        T_loc = K.empty(ng, w)
        T_all = K.empty(self.n, W)  # Y^T H, block by block (replicated after each allgather)
        for i in range(1, rp.p + 1):
            T = T_all[:, (i - 1) * w:i * w]
            K.spmm_t(self.Y_c, H[:, (i - 1) * w:i * w], out=T_loc)
            self.gather_n(T_loc, out=T)
            K.spmm(self.Y_r, T, out=H_loc)
            self.gather_m(H_loc, out=H[:, i * w:(i + 1) * w])
            normalise(i)
        if spec and not np.all(K.to_host(status).reshape(-1, 4)[:, 0] == -1.0):
            return self.bki(rp, allow_fallback, _speculate=False)
        self._passes = []
        X_loc = H[self.r0:self.r1]
        try:
            Q_loc = self._orth_rows(X_loc)
        except RankDeficiencyError as exc:
            self._passes = None
            fb.fail(exc)
            Q = K.dense_svd(H)[0]
            return self._project_and_solve(Q, rp.k, fb), Q, fb.count
        # Y^T Q = (Y^T H) R_1^{-1} R_2^{-1} ... from the Krylov products (the
        # single-GPU route's reuse, rsvd.KRYLOV_REUSE), gated on kappa_F(H)
        chain = self._chain(X_loc, Q_loc) if _rsvd.KRYLOV_REUSE else None
        if chain is not None and chain[1][0] == 0.0:
            R1inv = chain[0][0]
            kappa = float(np.sqrt(np.sum(K.diag(chain[1][1])) * float(K.to_host(K.stats(R1inv))[0])))
            if len(_rsvd.REUSE_STATS["kappas"]) < 4096:
                _rsvd.REUSE_STATS["kappas"].append(kappa)
            if np.isfinite(kappa) and kappa <= _rsvd.KRYLOV_REUSE_KAPPA:
                _rsvd.REUSE_STATS["used"] += 1
                T_loc = K.empty(ng, w)
                K.spmm_t(self.Y_c, H[:, rp.p * w:W], out=T_loc)
                self.gather_n(T_loc, out=T_all[:, rp.p * w:W])
                Bt_loc = T_all[self.c0:self.c1]
                for Rinv in chain[0]:
                    Bt_loc = K.matmul(Bt_loc, Rinv, b_upper=True)
                self._passes = None
                res = self._project_and_solve(None, rp.k, fb, Bt_loc=Bt_loc, Q_loc=Q_loc)
                return res, _GatheredQ(self, Q_loc, W), fb.count
        if chain is not None:
            _rsvd.REUSE_STATS["kappa_gate"] += 1
        self._passes = None
        Q = self.gather_m(Q_loc, out=K.empty(self.m, W))
        res = self._project_and_solve(Q, rp.k, fb)
        return res, Q, fb.count

    def recycle_q(self, cached: Subspace, k: int) -> DevSvd:
        width = cached.width
        if k > width:
            raise ValueError(f"requested rank {k} exceeds cached subspace width {width}")
        if k == 0:
            return self._empty()
        return self._project_and_solve(cached.Q_dev, k, _Fallback(False, None))

    def recycle_u(self, U_prev_loc) -> DevSvd:
        K = self.K
        k = int(U_prev_loc.shape[1])
        if k == 0:
            return self._empty()
        U_full = self.gather_m(U_prev_loc)
        try:
            Bt_loc = K.spmm_t(self.Y_c, U_full, out=K.empty(self.c1 - self.c0, k))
            desc = np.arange(k - 1, -1, -1)
            S, V, Usm, cols = self._eig_svd(Bt_loc, desc)
        except RankDeficiencyError as exc:
            raise RankDeficiencyError(f"projection onto cached U lost rank ({exc}); refresh the subspace") from exc
        U = K.matmul(U_prev_loc, K.select_columns(V, cols))
        Sd = np.asarray(S[cols], dtype=np.float64)
        return DevSvd(U, K.vector(Sd), Usm, Sd)

    def dense_full(self):
        """Descending dense SVD of the current Y (replicated), local rows."""
        K = self.K
        D_loc = K.from_host(K.densify(self.Y_r))
        D = self.gather_m(D_loc)
        U, S, V = K.dense_svd(D)
        return U[self.r0:self.r1], S, V[self.c0:self.c1]

    def dense_truncated(self, k: int) -> DevSvd:
        U, S, V = self.dense_full()
        return DevSvd(U[:, :k], self.K.vector(S[:k]), V[:, :k], S[:k].copy())

    # width guard of RsvdParams.check_against reads .rows / .cols
    @property
    def rows(self):
        return self.m

    @property
    def cols(self):
        return self.n


class _GatheredQ:
    """A row-sharded basis whose allgather is deferred until a caller needs
    the full Q (a recycle_q, Subspace.Q): rsvd_bki's own projection uses only
    the local rows."""

    def __init__(self, eng, Q_loc, W):
        self.eng, self.Q_loc, self.W = eng, Q_loc, W

    @property
    def shape(self):
        return (self.eng.m, self.W)

    def materialize(self):
        return self.eng.gather_m(self.Q_loc, out=self.eng.K.empty(self.eng.m, self.W))


# ------------------------------------------------------------ public API

def svt_sharded(obs: ObservationSet, params, backend: str = "rsvd-bki", strategy: str = None,
                exchange: Exchange = None, kernels=None):
    """SVT over all ranks of the default process group (every rank calls it
    with the same obs / params); the result (factors gathered) is returned on
    every rank.  strategy defaults to params.strategy (svt_fast semantics)."""
    from .completion import _svt_loop

    eng = ShardedEngine(obs, exchange, kernels)
    res = _svt_loop(obs, params, backend, params.strategy if strategy is None else strategy, engine=eng)
    res.plan = eng.plan.describe()
    return res


def rsvd_bki_sharded(A: SparseMatrix, params: RsvdParams, allow_fallback: bool = False,
                     exchange: Exchange = None, kernels=None, engine: ShardedEngine = None):
    """rsvd_bki over ranks: (SvdResult gathered on every rank, Subspace)."""
    eng = engine if engine is not None else ShardedEngine.from_matrix(A, exchange, kernels)
    res, Q, nfb = eng.bki(params, allow_fallback)
    k = params.k
    U = eng.K.to_host(eng.gather_m(res.U)) if k else np.zeros((eng.m, 0))
    V = eng.K.to_host(eng.gather_n(res.V)) if k else np.zeros((eng.n, 0))
    return SvdResult(U, res.S_host.copy(), V, "descending"), Subspace(Q, "bki", params.p, nfb)
