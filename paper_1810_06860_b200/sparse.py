"""Fixed-pattern sparse storage on the device and the sparse kernels of the
SVT / rSVD path.

Drop-in for /root/reference/pkg/src/lowrank/sparse.py:28-328 (the pattern,
the products, the sampled product, the in-place update, the scaled norm, the
spectral-norm estimate, and the observation sets).  Differences are in where
the data lives, not in what is computed:

* The pattern is built on the host exactly like the reference (lexsort by
  (row, col), stable argsort for the transpose index: integer work, bit-exact)
  and mirrored once on the device as int32 CSR + CSC + the CSC->CSR
  permutation and its inverse.
* The values keep TWO device copies, CSR order and CSC order, so Y^T X never
  re-gathers A.data[perm] per call (sparse.py:166-169) and the fused SVT step
  writes both copies in the same pass.
* Work schedules ("items") split rows longer than SPLIT_CHUNK entries so
  Zipf-shaped rows do not serialize a warp; partial rows are summed in fixed
  slot order, so every product is deterministic.
* `.data` stays a host numpy buffer with a stable identity: after device-side
  updates it is refreshed in place on access.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native, device
from .errors import DataError

SPLIT_CHUNK = 512
# rows longer than SKEW_RATIO x the mean trigger a longest-first item schedule
# (cfg4 CSR w = 16: 517 -> 261 us; cfg2 CSR w = 110: 322 -> 307 us)
SKEW_RATIO = 1.25
_SPECTRAL_TOL = 1e-3
_SPECTRAL_MAX_ITERS = 200
_SPECTRAL_BATCH = 8


# enough work items to fill the GPU several times over: small patterns (cfg1:
# 1000 rows of 200 entries) split their rows into short chunks so a product is
# not a few hundred latency-bound row walks (cfg1 CSR w = 16: 28 -> ~8 us)
TARGET_ITEMS = 148 * 64
MIN_CHUNK = 32


def _chunk_for(indptr: np.ndarray) -> int:
    nnz = int(indptr[-1]) if indptr.size else 0
    c = nnz // TARGET_ITEMS
    return int(min(SPLIT_CHUNK, max(MIN_CHUNK, c)))


def _schedule(indptr: np.ndarray, chunk: int = None):
    """Work items {row, beg, end, slot} (int32 x4) and split rows
    {row, slot_beg, slot_end, 0}; (None, None, 0) for a balanced pattern with
    no long row.  Items are ordered longest first: the lane groups of a warp
    then walk items of similar length (Zipf-shaped rows otherwise leave most
    groups idle behind the longest one) and the grid-stride loop drains the
    long items early.  Order does not affect results: every item owns its
    output row or split slot, and split slots are summed in slot order."""
    if chunk is None:
        chunk = _chunk_for(indptr)
    lens = np.diff(indptr)
    longm = lens > chunk
    skewed = lens.size > 0 and lens.max() > SKEW_RATIO * max(lens.mean(), 1.0)
    if not longm.any() and not skewed:
        return None, None, 0
    m = lens.shape[0]
    per_row = np.where(longm, (lens + chunk - 1) // chunk, 1)
    total = int(per_row.sum())
    rows = np.repeat(np.arange(m, dtype=np.int64), per_row)
    first = np.cumsum(per_row) - per_row
    k = np.arange(total, dtype=np.int64) - np.repeat(first, per_row)
    beg = indptr[rows] + k * chunk
    end = np.minimum(beg + chunk, indptr[rows + 1])
    is_long = np.repeat(longm, per_row)
    slot = np.full(total, -1, dtype=np.int64)
    n_slots = int(is_long.sum())
    slot[is_long] = np.arange(n_slots)
    items = np.stack([rows, beg, end, slot], axis=1).astype(np.int32)
    items = items[np.argsort(-(end - beg), kind="stable")]
    long_rows = np.flatnonzero(longm)
    s_cnt = per_row[long_rows]
    s_beg = np.cumsum(s_cnt) - s_cnt
    splits = np.stack([long_rows, s_beg, s_beg + s_cnt, np.zeros_like(long_rows)], axis=1).astype(np.int32)
    return items, splits, n_slots


class _HostSide:
    """Host-prepared int32 arrays + schedule of one orientation (built once
    per pattern, like the reference's lazily cached transpose index)."""

    def __init__(self, ptr_host, idx_host, n_rows):
        self.rows = int(n_rows)
        self.ptr = np.ascontiguousarray(ptr_host, dtype=np.int32)
        self.idx = np.ascontiguousarray(idx_host, dtype=np.int32)
        items, splits, n_slots = _schedule(np.asarray(ptr_host, dtype=np.int64))
        self.items = None if items is None else np.ascontiguousarray(items.ravel())
        self.splits = None if splits is None else np.ascontiguousarray(splits.ravel())
        self.n_items = self.rows if items is None else int(items.shape[0])
        self.n_splits = 0 if splits is None else int(splits.shape[0])
        self.n_slots = n_slots


class _Side:
    """One compressed orientation of the pattern on the device."""

    def __init__(self, hs: _HostSide = None, *, rows=None, ptr=None, idx=None, sched=None):
        if hs is not None:
            self.rows = hs.rows
            self.ptr = device.int_buffer(hs.ptr)
            self.idx = device.int_buffer(hs.idx)
            items, splits = hs.items, hs.splits
            self.n_items, self.n_splits, self.n_slots = hs.n_items, hs.n_splits, hs.n_slots
        else:  # built on the device; only the work schedule comes from the host
            self.rows, self.ptr, self.idx = rows, ptr, idx
            items, splits, n_slots = sched
            self.n_items = rows if items is None else int(items.shape[0])
            self.n_splits = 0 if splits is None else int(splits.shape[0])
            self.n_slots = n_slots
            items = None if items is None else items.ravel()
            splits = None if splits is None else splits.ravel()
        self.items = None if items is None else device.int_buffer(items)
        self.splits = None if splits is None else device.int_buffer(splits)
        self.counts_ptr = None  # the other orientation's offsets: their differences count this side's indices
        self._hot = False  # not examined yet; None: the pattern is not skewed enough

    def hot(self):
        """Hot-row encoding of this side's index stream for lr_spmm_hot_f64,
        built on the device once per pattern: (idx_hot, order, hot_max,
        share) with share[h - 1] = the fraction of stored entries whose index
        is among the h most frequent; None when staging the most frequent
        rows would serve less than HOT_MIN_SHARE of the gathers (uniform
        patterns: cfg2, cfg5)."""
        if self._hot is not False:
            return self._hot
        self._hot = None
        nnz = int(self.idx.numel())
        if not HOT_ROWS or self.counts_ptr is None or nnz < HOT_MIN_NNZ:
            return None
        cp = self.counts_ptr
        n_idx = int(cp.numel()) - 1
        hmax = min(int(_native.load().lr_spmm_hot_rows_max()), n_idx)
        if hmax < 32:
            return None
        cnt = (cp[1:] - cp[:-1]).to(torch.int64)
        # most frequent first, ties to the smaller index
        key = cnt * n_idx + (n_idx - 1 - torch.arange(n_idx, device=cnt.device, dtype=torch.int64))
        top = torch.topk(key, hmax, sorted=True).indices
        share = (torch.cumsum(cnt[top], 0).to(torch.float64) / max(nnz, 1)).cpu().numpy()
        if share[min(hmax, HOT_PROBE_ROWS) - 1] < HOT_MIN_SHARE:
            return None
        rank = torch.full((n_idx,), -1, dtype=torch.int32, device=cnt.device)
        rank[top] = torch.arange(hmax, device=cnt.device, dtype=torch.int32)
        idx_hot = torch.empty_like(self.idx)
        step = 1 << 24  # bounded temporaries
        for b in range(0, nnz, step):
            seg = self.idx[b:b + step]
            r = rank[seg.long()]
            idx_hot[b:b + step] = torch.where(r >= 0, -(r + 1), seg)
        self._hot = (idx_hot, top.to(torch.int32).contiguous(), hmax, share)
        return self._hot


# Shared-memory staging of the most frequent block rows (lr_spmm_hot_f64;
# north_star (1) "shared-memory/TMA staging of block rows"): opt-in
# (LR_SPMM_HOT=1).  Bit-identical to the plain kernel, but measured 2-3x
# SLOWER on cfg4 (profiles/r02ab_spmm_hot_probe.txt, r02ab_ncu_spmm_hot22.txt):
# the 1280 rows that fit shared memory at w = 22 serve only 39 % of the
# gathers (columns; 34 % for rows), every batch of 8 gathers still waits for
# its slowest L2 round trip (the kernel is latency-bound, not bandwidth-bound),
# the shared-memory carve-out leaves 28 KB of L1 (hit rate 22 % -> 2 %) and the
# two-source addressing nearly doubles the instruction count.  When enabled it
# is used when the HOT_PROBE_ROWS most frequent indices of a side carry at
# least HOT_MIN_SHARE of its stored entries and, per product, when the rows
# that fit shared memory at that width still do.
HOT_ROWS = __import__("os").environ.get("LR_SPMM_HOT", "0") == "1"
HOT_MIN_SHARE = float(__import__("os").environ.get("LR_SPMM_HOT_SHARE", "0.25"))
HOT_PROBE_ROWS = 1024
HOT_MIN_NNZ = 1 << 20
_HOT_SMEM_BYTES = 220 * 1024


class _HostPrep:
    """Host side of a pattern's upload: the CSR arrays as int32 and their
    work schedule (built once per pattern; pinned by SparseMatrix.pin_memory).
    The CSC side is derived on the device (lr_csr_transpose_i32)."""

    def pin(self) -> None:
        """Move every upload source into page-locked memory."""
        for name in ("ptr", "idx", "items", "splits"):
            a = getattr(self.csr, name)
            if a is not None:
                setattr(self.csr, name, device.pinned_copy(a))
        if self.csc_sched is not None:
            items, splits, n_slots = self.csc_sched
            self.csc_sched = (None if items is None else device.pinned_copy(items),
                              None if splits is None else device.pinned_copy(splits), n_slots)

    def __init__(self, A: "SparseMatrix"):
        self.csr = _HostSide(A.indptr, A.indices, A.rows)
        self.csc_sched = None  # (items, splits, n_slots) of the CSC side, from the device-built offsets


def _device_transpose(csr: _Side, m: int, n: int, nnz: int):
    """CSC structure (t_ptr, t_idx, perm, inv_perm) of a device CSR pattern,
    bit-exact with the host's stable argsort (sparse.py:129-139)."""
    import torch

    dev = device.require_cuda()
    i32 = torch.int32
    t_ptr = torch.empty(n + 1, dtype=i32, device=dev)
    t_idx = torch.empty(max(nnz, 1), dtype=i32, device=dev)
    perm = torch.empty(max(nnz, 1), dtype=i32, device=dev)
    inv = torch.empty(max(nnz, 1), dtype=i32, device=dev)
    ws = int(_native.load().lr_csr_transpose_workspace_ints(m, n))
    work = torch.empty(ws, dtype=i32, device=dev)
    _native.call("lr_csr_transpose_i32", m, n, nnz, device.ptr(csr.ptr), device.ptr(csr.idx), device.ptr(t_ptr),
                 device.ptr(t_idx), device.ptr(perm), device.ptr(inv), device.ptr(work), ws, device.stream())
    return t_ptr, t_idx, perm, inv


class DevicePattern:
    """CSR + CSC structure of one pattern on the device (shared by every
    matrix with that pattern, e.g. Y and P_Phi(M) in the SVT loop).  Only the
    CSR arrays are uploaded; the transpose index is built on the device and
    just the n+1 CSC offsets come back for the host-side work schedule."""

    def __init__(self, A: "SparseMatrix", prefetch_values=None):
        self.shape = (A.rows, A.cols)
        self.nnz = A.nnz
        if A._dev_csr is not None:  # built on the device: only the schedule comes from the host
            hp = A._host_prep_dev()
            self.csr = _Side(rows=A.rows, ptr=A._dev_csr[0], idx=A._dev_csr[1], sched=hp.csr_sched)
        else:
            hp = A._host_prep()
            self.csr = _Side(hp.csr)
        # the values' upload (side stream) overlaps the device transpose below
        self._prefetch = None
        if prefetch_values is not None and self.nnz:
            vc, done = device.f64_upload_async(prefetch_values)
            self._prefetch = (prefetch_values, vc, done)
        t_ptr, t_idx, self.perm, self.inv_perm = _device_transpose(self.csr, A.rows, A.cols, A.nnz)
        if hp.csc_sched is None:  # first upload of this pattern: offsets come back once
            hp.csc_sched = _schedule(device.to_host(t_ptr).astype(np.int64))
        self.csc = _Side(rows=A.cols, ptr=t_ptr, idx=t_idx, sched=hp.csc_sched)
        self.csr.counts_ptr, self.csc.counts_ptr = self.csc.ptr, self.csr.ptr

    def tile_rows(self):
        """Row of the first slot of every flat SVT tile (lr_svt_tile_rows_i32),
        built on the device once per pattern."""
        tr = getattr(self, "_tile_rows", None)
        if tr is None:
            lib = _native.load()
            n_tiles = int(lib.lr_svt_tile_count(self.nnz))
            tr = torch.empty(max(n_tiles, 1), dtype=torch.int32, device=device.require_cuda())
            if n_tiles:
                _native.call("lr_svt_tile_rows_i32", device.ptr(self.csr.ptr), self.csr.rows, self.nnz,
                             device.ptr(tr), device.stream())
            self._tile_rows = tr
        return tr

    def values_from_device(self, vc):
        """(csr, csc) device value copies from a device CSR-order vector."""
        vt = device.vector(self.nnz)
        if self.nnz:
            _native.call("lr_gather_f64", device.ptr(vc), device.ptr(self.perm), device.ptr(vt), self.nnz,
                         device.stream())
        return vc, vt

    def values(self, host_vals: np.ndarray):
        """(csr, csc) device value copies of host values in CSR order."""
        pre = self._prefetch
        if pre is not None and pre[0] is host_vals:
            self._prefetch = None
            vc = pre[1]
            torch.cuda.current_stream().wait_event(pre[2])
        else:
            vc = device.f64_buffer(host_vals)
        vt = device.vector(self.nnz)
        if self.nnz:
            _native.call("lr_gather_f64", device.ptr(vc), device.ptr(self.perm), device.ptr(vt),
                         self.nnz, device.stream())
        return vc, vt

class SparseMatrix:
    """CSR matrix with an immutable pattern (sparse.py:28-150 contract).

    rows, cols; indptr / indices int64 host arrays (columns strictly
    increasing within a row); data float64 (explicit zeros are legal).  The
    sanctioned mutation is `update_pattern_values`.
    """

    _dev_csr = None  # (ptr, idx int32, values) when the pattern was built on the device

    def __init__(self, rows: int, cols: int, indptr, indices, data):
        self.rows = int(rows)
        self.cols = int(cols)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self._indices = np.ascontiguousarray(indices, dtype=np.int64)
        self._data = np.ascontiguousarray(data, dtype=np.float64)
        self._validate()
        self._tperm = self._t_indptr = self._t_indices = self._coo_rows = None
        self._pattern = None  # DevicePattern (shared structure)
        self._dvals = None  # (csr, csc) device values
        self._host_stale = False
        self._csc_stale = False  # CSR copy updated in place; CSC copy refreshed on demand

    @property
    def indices(self) -> np.ndarray:
        """Column indices (int64, host); a device-built pattern downloads them
        on first access."""
        if self._indices is None:
            self._indices = device.to_host(self._dev_csr[1]).astype(np.int64)
        return self._indices

    @indices.setter
    def indices(self, value):
        self._indices = value

    @classmethod
    def from_coo_device(cls, rows: int, cols: int, i, j, v, split=None, tag: int = 0,
                        range_msg=("coordinate out of range", "coordinate out of range"),
                        dup_msg=None, uploaded=None) -> "SparseMatrix":
        """from_coo on the device (lr_coo_to_csr_i32: bounds, duplicates, row
        buckets + per-row column sort -- the same CSR as the host lexsort, bit
        for bit).  The host keeps only indptr (the work schedule needs it);
        indices and values come back on access.  With `split` (uint8 tags),
        only the entries tagged `tag` are used (ObservationSet.train_matrix)."""
        import ctypes

        rows, cols = int(rows), int(cols)
        if rows < 1 or cols < 1:
            raise DataError(f"matrix dims must be positive, got {rows}x{cols}")
        count = int(np.asarray(i).shape[0])
        if not (np.asarray(j).shape[0] == np.asarray(v).shape[0] == count):
            raise DataError("coordinate arrays must be 1-D and equal length")
        if count >= (1 << 31) - 1:
            return cls.from_coo(rows, cols, *_select(i, j, v, split, tag))
        dev = device.require_cuda()
        st = device.stream()
        if uploaded is None:
            uploaded = _upload_coo(i, j, v, split)
        di, dj, dv, ds = uploaded
        i32 = torch.int32
        ptr = torch.empty(rows + 1, dtype=i32, device=dev)
        col = torch.empty(max(count, 1), dtype=i32, device=dev)
        src = torch.empty(max(count, 1), dtype=i32, device=dev)
        vals = torch.empty(max(count, 1), dtype=torch.float64, device=dev)
        lib = _native.load()
        ws = int(lib.lr_coo_to_csr_workspace_ints(rows, count))
        work = torch.empty(max(ws, 1), dtype=i32, device=dev)
        status = (ctypes.c_int * 3)()
        _native.call("lr_coo_to_csr_i32", rows, cols, count, device.ptr(di), device.ptr(dj), device.ptr(ds),
                     int(tag), device.ptr(dv), device.ptr(ptr), device.ptr(col), device.ptr(src), device.ptr(vals),
                     device.ptr(work), ws, ctypes.byref(status), st)
        if status[0] in (1, 3):
            raise DataError(range_msg[0] if status[0] == 1 else range_msg[1])
        if status[0] == 2:
            raise DataError("matrix values must be finite")
        nnz = int(status[2])
        indptr = device.to_host(ptr).astype(np.int64)
        if status[1] >= 0:
            if dup_msg is not None:
                raise DataError(dup_msg)
            p = int(status[1])
            r = int(np.searchsorted(indptr, p, side="right") - 1)
            c = int(device.to_host(col[p:p + 1])[0])
            raise DataError(f"duplicate entry at ({r}, {c})")
        out = cls.__new__(cls)
        out.rows, out.cols = rows, cols
        out.indptr = indptr
        out._indices = None
        out._data = np.empty(nnz)
        out._tperm = out._t_indptr = out._t_indices = out._coo_rows = None
        out._pattern = None
        out._dvals = None
        out._host_stale = True  # host values download on access
        out._csc_stale = False
        out._dev_csr = (ptr, col[:nnz], vals[:nnz])
        return out

    @classmethod
    def from_device_csr(cls, rows: int, cols: int, indptr_host, ptr, idx, vals) -> "SparseMatrix":
        """A matrix whose CSR arrays already sit on the device (int32 ptr of
        rows + 1 offsets, int32 idx, float64 vals: e.g. a row or column block
        cut out of a device-built CSR, shards.py): the host keeps indptr (the
        work schedule needs it); indices and values come back on access.  The
        arrays are trusted (they come from a validated matrix)."""
        out = cls.__new__(cls)
        out.rows, out.cols = int(rows), int(cols)
        out.indptr = np.ascontiguousarray(indptr_host, dtype=np.int64)
        nnz = int(out.indptr[-1]) if out.indptr.size else 0
        out._indices = None
        out._data = np.empty(nnz)
        out._tperm = out._t_indptr = out._t_indices = out._coo_rows = None
        out._pattern = None
        out._dvals = None
        out._host_stale = True
        out._csc_stale = False
        out._dev_csr = (ptr, idx, vals)
        return out

    # ------------------------------------------------------------ checks
    def _validate(self) -> None:
        if self.rows < 1 or self.cols < 1:
            raise DataError(f"matrix dims must be positive, got {self.rows}x{self.cols}")
        if self.indptr.shape != (self.rows + 1,):
            raise DataError(f"indptr length {self.indptr.shape[0]} != rows + 1 = {self.rows + 1}")
        if self.indptr[0] != 0 or np.any(self.indptr[1:] < self.indptr[:-1]):
            raise DataError("row offsets must start at 0 and be monotone")
        nnz = int(self.indptr[-1])
        if self.indices.shape != (nnz,) or self._data.shape != (nnz,):
            raise DataError("indices/data length must equal last row offset")
        if nnz:
            if self.indices.min() < 0 or self.indices.max() >= self.cols:
                raise DataError("column index out of range")
            step_ok = np.ones(max(nnz - 1, 0), dtype=bool)
            inner = np.diff(self.indices) > 0
            row_start = self.indptr[1:-1]
            row_start = row_start[(row_start > 0) & (row_start < nnz)]
            at_break = np.zeros(max(nnz - 1, 0), dtype=bool)
            at_break[row_start - 1] = True
            step_ok = inner | at_break
            if not step_ok.all():
                raise DataError("column indices must strictly increase within a row")
        if not np.isfinite(self._data).all():
            raise DataError("matrix values must be finite")

    # ------------------------------------------------------ construction
    @classmethod
    def from_coo(cls, rows: int, cols: int, i, j, v) -> "SparseMatrix":
        """Coordinate triples -> CSR (lexsort by row then column); duplicates
        raise DataError (sparse.py:84-104)."""
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        if not (i.shape == j.shape == v.shape) or i.ndim != 1:
            raise DataError("coordinate arrays must be 1-D and equal length")
        if i.size and (i.min() < 0 or i.max() >= rows or j.min() < 0 or j.max() >= cols):
            raise DataError("coordinate out of range")
        order = np.lexsort((j, i))
        i, j, v = i[order], j[order], v[order]
        if i.size > 1:
            dup = (i[1:] == i[:-1]) & (j[1:] == j[:-1])
            if dup.any():
                k = int(np.argmax(dup))
                raise DataError(f"duplicate entry at ({i[k]}, {j[k]})")
        indptr = np.zeros(rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(i, minlength=rows), out=indptr[1:])
        return cls(rows, cols, indptr, j, v)

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        ar = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), ar, np.ones(n))

    # --------------------------------------------------------- structure
    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def data(self) -> np.ndarray:
        if self._host_stale:
            src = self._dvals[0] if self._dvals is not None else self._dev_csr[2]
            self._data[...] = device.to_host(src)
            self._host_stale = False
        return self._data

    def coo_rows(self) -> np.ndarray:
        if self._coo_rows is None:
            self._coo_rows = np.repeat(np.arange(self.rows, dtype=np.int64), np.diff(self.indptr))
        return self._coo_rows

    def _transpose_index(self):
        # stable sort by column keeps rows ascending inside each column
        if self._tperm is None:
            self._tperm = np.argsort(self.indices, kind="stable")
            t_indptr = np.zeros(self.cols + 1, dtype=np.int64)
            np.cumsum(np.bincount(self.indices, minlength=self.cols), out=t_indptr[1:])
            self._t_indptr = t_indptr
            self._t_indices = self.coo_rows()[self._tperm]
        return self._tperm, self._t_indptr, self._t_indices

    def densify(self) -> np.ndarray:
        out = np.zeros(self.shape)
        out[self.coo_rows(), self.indices] = self.data
        return out

    # ------------------------------------------------------------ device
    def _host_prep_dev(self):
        """Host side of a device-built pattern: the CSR work schedule (from
        indptr) and the CSC schedule cache."""
        hp = getattr(self, "_hprep_dev", None)
        if hp is None:
            hp = self._hprep_dev = type("_DevPrep", (), {})()
            hp.csr_sched = _schedule(self.indptr)
            hp.csc_sched = None
        return hp

    def _host_prep(self) -> _HostPrep:
        if getattr(self, "_hprep", None) is None:
            self._hprep = _HostPrep(self)
        return self._hprep

    def pattern(self) -> DevicePattern:
        if self._pattern is None:
            # first device use: the values ride along (uploaded while the
            # transpose index is built) unless they are already resident
            pre = self._data if (self._dvals is None and not self._host_stale and self._dev_csr is None) else None
            self._pattern = DevicePattern(self, prefetch_values=pre)
        return self._pattern

    def pin_memory(self) -> "SparseMatrix":
        """Keep the host side (values and the prepared CSR/CSC index arrays)
        in page-locked memory, so every (re-)upload of this matrix is a
        direct DMA.  Returns self."""
        if self._host_stale:
            _ = self.data
        self._data = device.pinned_copy(self._data)
        self._host_prep().pin()
        return self

    def drop_device(self) -> None:
        """Release the device mirror (pattern and values); host data stay."""
        if self._host_stale:
            _ = self.data
        self._pattern = None
        self._dvals = None

    def share_pattern(self, other: "SparseMatrix") -> None:
        """Reuse other's device structure (same indptr/indices objects)."""
        if other._pattern is not None:
            self._pattern = other._pattern
            self._tperm, self._t_indptr, self._t_indices = other._tperm, other._t_indptr, other._t_indices
            self._coo_rows = other._coo_rows
            self._hprep = getattr(other, "_hprep", None)

    def device_values(self):
        """(csr, csc) device value vectors, created from the host data once.
        After an in-place update of the CSR copy alone (the fused SVT step,
        `mark_csc_stale`) the CSC copy is refreshed here by one gather pass
        (csc[s] = csr[perm[s]]: coalesced perm read and store, one random 8-byte
        read per entry) before anything reads it."""
        if self._dvals is None:
            if self._dev_csr is not None and self._host_stale:
                self._dvals = self.pattern().values_from_device(self._dev_csr[2])
            else:
                self._dvals = self.pattern().values(self._data)
            self._csc_stale = False
        elif self._csc_stale:
            vc, vt = self._dvals
            if self.nnz:
                _native.call("lr_gather_f64", device.ptr(vc), device.ptr(self.pattern().perm), device.ptr(vt),
                             self.nnz, device.stream(), meta={"nnz": self.nnz})
            self._csc_stale = False
        return self._dvals

    def scaled_on_device(self, scale: float) -> "SparseMatrix":
        """SparseMatrix(rows, cols, indptr, indices, scale * data) sharing this
        matrix's pattern, with the product formed on the device from this
        matrix's two resident value copies (one IEEE multiply per entry: the
        same bits as the host product; completion.py:335's Y = c delta P(M)).
        The host copy of the new values is materialised only on access.  The
        constructor's finiteness check holds iff scale * max|data| is finite
        (rounding is monotone), so it is decided from one cached scalar."""
        scale = float(scale)
        mx = getattr(self, "_maxabs", None)
        if mx is None:  # max |data| from the resident CSR copy (one device reduction)
            mx = float(device.to_host(_stats(self.device_values()[0], self.nnz, 1, 1))[1]) if self.nnz else 0.0
            self._maxabs = mx
        if not (np.isfinite(scale) and np.isfinite(scale * mx)):
            raise DataError("matrix values must be finite")
        out = SparseMatrix.__new__(SparseMatrix)
        out.rows, out.cols = self.rows, self.cols
        out.indptr, out._indices = self.indptr, self._indices
        if self._dev_csr is not None:  # indices stay on the device until asked for
            out._dev_csr = (self._dev_csr[0], self._dev_csr[1], None)
            out._hprep_dev = self._host_prep_dev()
        out._data = np.empty(self.nnz)
        out._tperm = out._t_indptr = out._t_indices = out._coo_rows = None
        out._pattern = None
        out._host_stale = False
        out._csc_stale = False
        self.pattern()
        out.share_pattern(self)
        src = self.device_values()
        sv = device.f64_buffer(np.array([scale]))
        dst = []
        for v in src:
            d = device.vector(self.nnz)
            if self.nnz:
                _native.call("lr_scale_columns_f64", device.ptr(v), 1, self.nnz, None, 1, device.ptr(sv), 0,
                             device.ptr(d), 1, device.stream())
            dst.append(d)
        out._dvals = (dst[0], dst[1])
        out._host_stale = True
        return out

    def device_values_csr(self):
        """The CSR device value vector (no CSC refresh)."""
        if self._dvals is None:
            self.device_values()
        return self._dvals[0]

    def mark_csc_stale(self):
        self._csc_stale = True

    def device_values32(self):
        """(csr, csc) fp32 copies of the device values (fp32 mode), rounded
        from the fp64 copies once per value state."""
        vals = self.device_values()
        cached = getattr(self, "_dvals32", None)
        if cached is None or cached[0] is not vals:
            cached = (vals, device.to_f32(vals[0]), device.to_f32(vals[1]))
            self._dvals32 = cached
        return cached[1], cached[2]


# --------------------------------------------------------------- kernels

def _upload_coo(i, j, v, split=None):
    """Device copies of COO triples (+ split tags), asynchronous from pinned
    host arrays."""
    dev = device.require_cuda()
    di = device.upload_async_i64(i)
    dj = device.upload_async_i64(j)
    dv = device.f64_buffer(np.asarray(v, dtype=np.float64))
    ds = None
    if split is not None:
        ds = torch.from_numpy(np.ascontiguousarray(split, dtype=np.uint8)).to(dev, non_blocking=True)
    return di, dj, dv, ds


def _select(i, j, v, split, tag):
    if split is None:
        return i, j, v
    sel = np.asarray(split) == tag
    return np.asarray(i)[sel], np.asarray(j)[sel], np.asarray(v)[sel]


def _spmm_side(side: _Side, vals, X, out=None):
    rows_out = side.rows
    w = int(X.shape[1])
    if out is None:
        out = device.empty(rows_out, w)
    scratch = None
    if side.n_splits:
        scratch = device.arena().get("spmm_scratch", side.n_slots * max(w, 1) + 2)
    hot = side.hot() if w >= 2 else None
    if hot is not None:
        # rows of a <= 128-column chunk that fit shared memory, and the share of the gathers they serve
        fit = _HOT_SMEM_BYTES // (((min(w, 128) + 1) // 2) * 16)
        if fit < 32 or hot[3][min(fit, hot[2]) - 1] < HOT_MIN_SHARE:
            hot = None
    if hot is not None:
        nbuf = int(_native.load().lr_spmm_hot_buf_doubles())
        hbuf = device.arena().get("spmm_hot_buf", nbuf)
        _native.call("lr_spmm_hot_f64", device.ptr(side.ptr), device.ptr(side.idx), device.ptr(hot[0]),
                     device.ptr(hot[1]), hot[2], device.ptr(hbuf), nbuf, device.ptr(vals), side.rows,
                     device.ptr(side.items), side.n_items if side.items is not None else side.rows,
                     device.ptr(side.splits), side.n_splits, device.ptr(X), device.ld(X), w,
                     device.ptr(out), device.ld(out), device.ptr(scratch), device.stream(),
                     meta={"nnz": int(side.idx.numel()), "rows": side.rows, "cols": int(X.shape[0]), "w": w})
        return out
    _native.call("lr_spmm_f64", device.ptr(side.ptr), device.ptr(side.idx), device.ptr(vals), side.rows,
                 device.ptr(side.items), side.n_items if side.items is not None else side.rows,
                 device.ptr(side.splits), side.n_splits, device.ptr(X), device.ld(X), w,
                 device.ptr(out), device.ld(out), device.ptr(scratch), device.stream(),
                 meta={"nnz": int(side.idx.numel()), "rows": side.rows, "cols": int(X.shape[0]), "w": w})
    return out


def _spmm_side32(side: _Side, vals32, X32, out=None):
    rows_out = side.rows
    w = int(X32.shape[1])
    if out is None:
        out = device.empty32(rows_out, w)
    scratch = None
    if side.n_splits:  # fp32 partial rows fit the fp64 arena buffer
        scratch = device.arena().get("spmm_scratch", (side.n_slots * max(w, 1) + 3) // 2 + 2)
    _native.call("lr_spmm_f32", device.ptr(side.ptr), device.ptr(side.idx), device.ptr(vals32), side.rows,
                 device.ptr(side.items), side.n_items if side.items is not None else side.rows,
                 device.ptr(side.splits), side.n_splits, device.ptr(X32), device.ld(X32), w,
                 device.ptr(out), device.ld(out), device.ptr(scratch), device.stream(),
                 meta={"nnz": int(side.idx.numel()), "rows": side.rows, "cols": int(X32.shape[0]), "w": w,
                       "bytes_per_value": 4})
    return out


def spmm_dev32(A: SparseMatrix, X32, out=None):
    """fp32 mode: Y @ X with fp32 values and fp32 blocks (w >= 2)."""
    return _spmm_side32(A.pattern().csr, A.device_values32()[0], X32, out)


def spmm_t_dev32(A: SparseMatrix, H32, out=None):
    """fp32 mode: Y^T @ H with fp32 values and fp32 blocks (w >= 2)."""
    return _spmm_side32(A.pattern().csc, A.device_values32()[1], H32, out)


def spmm_dev(A: SparseMatrix, X, out=None):
    """Device Y @ X (X: n x w device block) -> m x w device block."""
    return _spmm_side(A.pattern().csr, A.device_values()[0], X, out)


def spmm_t_dev(A: SparseMatrix, H, out=None):
    """Device Y^T @ H (H: m x w device block) -> n x w device block."""
    return _spmm_side(A.pattern().csc, A.device_values()[1], H, out)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def spmm(A: SparseMatrix, X):
    """A @ X (sparse.py:153-158).  numpy in -> numpy out; CUDA tensor in ->
    CUDA tensor out."""
    if X is None or np.ndim(X) != 2 or A.cols != X.shape[0]:
        shp = getattr(X, "shape", None)
        raise ValueError(f"spmm dimension mismatch: {A.shape} @ {shp}")
    out = spmm_dev(A, device.to_device(X))
    return out if _is_torch(X) else device.to_host(out)


def spmm_t(A: SparseMatrix, X):
    """A.T @ X via the persistent CSC copy (sparse.py:161-170)."""
    if X is None or np.ndim(X) != 2 or A.rows != X.shape[0]:
        shp = getattr(X, "shape", None)
        raise ValueError(f"spmm_t dimension mismatch: {A.shape}^T @ {shp}")
    out = spmm_t_dev(A, device.to_device(X))
    return out if _is_torch(X) else device.to_host(out)


# SDDMM / fused SVT step kernel family: "items" (default: a G-lane group per
# row / row chunk, line-aligned V gathers, U * S of the row in registers;
# lr_sddmm_f64 / lr_svt_step_f64) or "flat" (tiles of consecutive CSR slots,
# one warp each; lr_*_flat_f64)
SVT_KERNEL = "items"


def project_pattern_dev(U, S, V, pattern: SparseMatrix, out=None):
    dp = pattern.pattern()
    r = int(S.shape[0])
    if out is None:
        out = device.vector(pattern.nnz)
    if pattern.nnz == 0:
        return out
    if r == 0:
        _native.call("lr_fill_f64", device.ptr(out), 1, pattern.nnz, 1, 0.0, device.stream())
        return out
    if SVT_KERNEL == "flat":
        _native.call("lr_sddmm_flat_f64", device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), dp.csr.rows,
                     pattern.nnz, device.ptr(dp.tile_rows()), device.ptr(U), device.ld(U), device.ptr(S),
                     device.ptr(V), device.ld(V), r, device.ptr(out), device.stream())
        return out
    _native.call("lr_sddmm_f64", device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), dp.csr.rows,
                 device.ptr(dp.csr.items), dp.csr.n_items, device.ptr(U), device.ld(U), device.ptr(S),
                 device.ptr(V), device.ld(V), r, device.ptr(out), device.stream())
    return out


def _vec_dev(x):
    import torch

    if isinstance(x, torch.Tensor) and x.device.type == "cuda":
        return x.to(torch.float64).contiguous()
    return device.f64_buffer(np.asarray(x, dtype=np.float64).ravel())


def project_pattern(U, S, V, pattern: SparseMatrix):
    """Entries of U diag(S) V^T on the pattern, CSR order (sparse.py:173-191)."""
    if U.shape[0] != pattern.rows or V.shape[0] != pattern.cols:
        raise ValueError("factor dims do not match pattern dims")
    if U.shape[1] != S.shape[0] or V.shape[1] != S.shape[0]:
        raise ValueError("factor rank mismatch")
    r = int(S.shape[0])
    Ud = device.to_device(U) if r else None
    Vd = device.to_device(V) if r else None
    out = project_pattern_dev(Ud, _vec_dev(S), Vd, pattern)
    return out if _is_torch(U) else device.to_host(out)


def project_observed(U, S, V, obs: "ObservationSet"):
    """Sampled entries of U diag(S) V^T on the train split of obs."""
    if U.shape[0] != obs.m or V.shape[0] != obs.n:
        raise ValueError("factor dims do not match observation dims")
    if U.shape[1] != S.shape[0] or V.shape[1] != S.shape[0]:
        raise ValueError("factor rank mismatch")
    mask = obs.split == ObservationSet.TRAIN
    return sample_at(U, S, V, obs.rows[mask], obs.cols[mask])


def sample_at(U, S, V, rows, cols):
    """U diag(S) V^T at arbitrary (rows, cols), in the given order."""
    n_e = int(rows.shape[0])
    r = int(S.shape[0])
    out = device.vector(n_e)
    if n_e == 0:
        return device.to_host(out)
    if r == 0:
        return np.zeros(n_e)
    # every entry is its own "row" of a pattern with rows -> U rows via items
    items = np.stack([np.asarray(rows, np.int64), np.arange(n_e), np.arange(n_e) + 1,
                      np.full(n_e, -1)], axis=1).astype(np.int32)
    d_items = device.int_buffer(items.ravel())
    d_idx = device.int_buffer(np.asarray(cols))
    Ud, Vd, Sd = device.to_device(U), device.to_device(V), _vec_dev(S)
    _native.call("lr_sddmm_f64", device.ptr(d_idx), device.ptr(d_idx), n_e, device.ptr(d_items), n_e,
                 device.ptr(Ud), device.ld(Ud), device.ptr(Sd), device.ptr(Vd), device.ld(Vd), r,
                 device.ptr(out), device.stream())
    return device.to_host(out)


def update_pattern_values(Y: SparseMatrix, delta_vals) -> SparseMatrix:
    """Y.data += delta_vals in place on the device (both value copies); the
    pattern and the host buffer identity are untouched (sparse.py:205-216)."""
    if tuple(np.shape(delta_vals)) != (Y.nnz,):
        raise ValueError(f"delta length {tuple(np.shape(delta_vals))} != nnz {Y.nnz}")
    vc, vt = Y.device_values()
    d = _vec_dev(delta_vals)
    _native.call("lr_pattern_axpy_f64", device.ptr(vc), device.ptr(vt), device.ptr(Y.pattern().inv_perm),
                 device.ptr(d), 1.0, Y.nnz, device.stream())
    Y._host_stale = True
    Y._dvals32 = None
    return Y


def _stats(x, rows, cols, ldx):
    part = device.arena().get("stats_partial", _native.load().lr_stats_partials() + 8)
    out = device.vector(3)
    _native.call("lr_block_stats_f64", device.ptr(x), rows, cols, ldx, device.ptr(part), device.ptr(out),
                 device.stream())
    return out


def frobenius_dev(x) -> float:
    """Scaled-safe Euclidean norm of a device vector/block (one sync)."""
    if x.dim() == 1:
        rows, cols, ldx = x.shape[0], 1, 1
    else:
        rows, cols, ldx = x.shape[0], x.shape[1], device.ld(x)
    if rows * cols == 0:
        return 0.0
    s = device.to_host(_stats(x, rows, cols, ldx))
    sumsq, big = float(s[0]), float(s[1])
    if big == 0.0:
        return 0.0
    if np.isfinite(sumsq) and 1e-150 < big < 1e150:
        return float(np.sqrt(sumsq))
    # rescale on the device when squares would over/underflow
    y = device.empty(rows, cols)
    scale = device.f64_buffer(np.full(max(cols, 1), big))
    _native.call("lr_scale_columns_f64", device.ptr(x), ldx, rows, None, cols, device.ptr(scale), 1,
                 device.ptr(y), device.ld(y), device.stream())
    s2 = device.to_host(_stats(y, rows, cols, device.ld(y)))
    return float(big * np.sqrt(s2[0]))


def frobenius(values) -> float:
    """Euclidean norm with overflow-safe scaling (sparse.py:219-228)."""
    if _is_torch(values):
        return frobenius_dev(values.reshape(-1))
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        return 0.0
    return frobenius_dev(device.f64_buffer(v))


class PowerIteration:
    """Device state of the power iteration on A^T A (sparse.py:231-256):
    x = x0 / ||x0||; each `update(z)` with z = A^T A x records the estimate
    sqrt(x.z), the 1e-3 relative-agreement latch and x <- z / ||z||, all on
    the device, so the host polls `done()` only every few steps."""

    def __init__(self, x0_host: np.ndarray):
        n = int(np.asarray(x0_host).size)
        self.n = n
        # unit-stride (n, 1) views: the dot / power kernels treat them as flat vectors
        x = device.f64_buffer(np.asarray(x0_host, dtype=np.float64).ravel()).view(n, 1)
        self.part = device.arena().get("power_partial", 2 * 4096)
        nrm2 = device.vector(1)
        _native.call("lr_dot_f64", device.ptr(x), device.ptr(x), n, device.ptr(self.part), device.ptr(nrm2),
                     device.stream())
        nrm = float(np.sqrt(device.to_host(nrm2)[0]))
        inv = device.f64_buffer(np.array([nrm]))
        xs = device.vector(n).view(n, 1)
        _native.call("lr_scale_columns_f64", device.ptr(x), 1, n, None, 1, device.ptr(inv), 1,
                     device.ptr(xs), 1, device.stream())
        self.x = xs
        self.state = device.f64_buffer(np.zeros(6))

    def update(self, z) -> None:
        _native.call("lr_power_update_f64", device.ptr(self.x), device.ptr(z), self.n, _SPECTRAL_TOL,
                     device.ptr(self.state), device.ptr(self.part), device.stream())

    def done(self) -> bool:
        return device.to_host(self.state)[2] != 0.0

    def result(self) -> float:
        st = device.to_host(self.state)
        if st[4] != 0.0:
            return 0.0
        return float(max(st[0], st[1]))


def spectral_norm_est_dev(A: SparseMatrix, x0_host: np.ndarray) -> float:
    """Power iteration on A^T A from x0 (sparse.py:231-256): stop at 1e-3
    relative agreement or 200 steps; return the larger of the last two."""
    n, m = A.cols, A.rows
    pw = PowerIteration(x0_host)
    y = device.vector(m).view(m, 1)
    z = device.vector(n).view(n, 1)
    for it in range(_SPECTRAL_MAX_ITERS):
        if it and it % _SPECTRAL_BATCH == 0 and pw.done():
            break
        spmm_dev(A, pw.x, out=y)
        spmm_t_dev(A, y, out=z)
        pw.update(z)
    return pw.result()


def spectral_norm_est(A: SparseMatrix, rng) -> float:
    """Largest singular value estimate (sparse.py:231-256); the starting
    vector comes from rng.normal_pairs(A.cols) as in the reference."""
    if A.nnz < 1:
        raise ValueError("spectral norm estimate needs at least one stored entry")
    return spectral_norm_est_dev(A, rng.normal_pairs(A.cols))


class ObservationSet:
    """Split-tagged coordinate samples (sparse.py:259-328): TRAIN = 0,
    TEST = 1; duplicate cells within a split are rejected."""

    TRAIN = 0
    TEST = 1

    def __init__(self, m: int, n: int, rows, cols, values, split=None):
        self.m = int(m)
        self.n = int(n)
        self.rows = np.ascontiguousarray(rows, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if split is None:
            split = np.zeros(self.rows.shape[0], dtype=np.uint8)
        self.split = np.ascontiguousarray(split, dtype=np.uint8)
        self._validate()

    def _validate(self) -> None:
        if self.m < 1 or self.n < 1:
            raise DataError(f"observation dims must be positive, got {self.m}x{self.n}")
        cnt = self.rows.shape[0]
        if not (self.cols.shape[0] == self.values.shape[0] == self.split.shape[0] == cnt):
            raise DataError("observation arrays must have equal length")
        if cnt and device.cuda_ready() and cnt < (1 << 31) - 1:
            self._validate_device()
            return
        if cnt:
            if self.rows.min() < 0 or self.rows.max() >= self.m:
                raise DataError("observation row index out of range")
            if self.cols.min() < 0 or self.cols.max() >= self.n:
                raise DataError("observation col index out of range")
        if not np.isfinite(self.values).all():
            raise DataError("observation values must be finite")
        if np.any(self.split > 1):
            raise DataError("split tags must be 0 (train) or 1 (test)")
        for tag, name in ((self.TRAIN, "train"), (self.TEST, "test")):
            sel = self.split == tag
            key = self.rows[sel] * self.n + self.cols[sel]
            if key.size != np.unique(key).size:
                raise DataError(f"duplicate (row, col) within {name} split")

    def _validate_device(self) -> None:
        """The same checks, in the same order, with the duplicate search of
        each split on the device (lr_coo_to_csr_i32 over the split's cells:
        the host np.unique of ~20M keys costs seconds).  The train split's
        device CSR is kept for train_matrix()."""
        msgs = ("observation row index out of range", "observation col index out of range")
        if self.rows.min() < 0 or self.rows.max() >= self.m:
            raise DataError(msgs[0])
        if self.cols.min() < 0 or self.cols.max() >= self.n:
            raise DataError(msgs[1])
        if not np.isfinite(self.values).all():
            raise DataError("observation values must be finite")
        if np.any(self.split > 1):
            raise DataError("split tags must be 0 (train) or 1 (test)")
        up = _upload_coo(self.rows, self.cols, self.values, self.split)  # once for both splits
        self._train_dev = SparseMatrix.from_coo_device(self.m, self.n, self.rows, self.cols, self.values, self.split,
                                                       self.TRAIN, range_msg=msgs,
                                                       dup_msg="duplicate (row, col) within train split",
                                                       uploaded=up)
        if np.any(self.split == self.TEST):
            SparseMatrix.from_coo_device(self.m, self.n, self.rows, self.cols, self.values, self.split, self.TEST,
                                         range_msg=msgs, dup_msg="duplicate (row, col) within test split",
                                         uploaded=up)

    @property
    def count(self) -> int:
        return self.rows.shape[0]

    @property
    def train_count(self) -> int:
        return int(np.count_nonzero(self.split == self.TRAIN))

    @property
    def test_count(self) -> int:
        return int(np.count_nonzero(self.split == self.TEST))

    def subset(self, tag: int):
        sel = self.split == tag
        return self.rows[sel], self.cols[sel], self.values[sel]

    def train_matrix(self) -> SparseMatrix:
        """The train split as CSR: built on the device when one is present
        (SparseMatrix.from_coo_device: the host lexsort of ~20M cells costs
        seconds), else on the host."""
        pre = getattr(self, "_train_dev", None)
        if pre is not None:  # built by the device validation; hand it out once
            self._train_dev = None
            return pre
        if device.cuda_ready():
            return SparseMatrix.from_coo_device(self.m, self.n, self.rows, self.cols, self.values, self.split,
                                                self.TRAIN)
        r, c, v = self.subset(self.TRAIN)
        return SparseMatrix.from_coo(self.m, self.n, r, c, v)
