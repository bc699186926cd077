"""Device plumbing: CUDA availability, the working stream, padded dense
blocks and a reusable scratch arena.

Dense device blocks are torch float64 tensors viewed as (rows, cols) with
row stride `ld` >= cols (ld rounded up to an even count so rows are 16-byte
aligned for the double2 paths of the kernels).  torch owns every device
buffer; the native library never allocates.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

F64 = torch.float64
I32 = torch.int32

# host<->device traffic of this process, for the bench's e2e accounting
TRAFFIC = {"h2d": 0, "d2h": 0}


_READY = False
_DEVICES = {}


def cuda_ready() -> bool:
    """A CUDA device and the native library are present (the device paths
    of input preparation apply)."""
    if _READY:
        return True
    try:
        require_cuda()
        return True
    except (RuntimeError, ImportError):
        return False


def upload_async_i64(a) -> torch.Tensor:
    """int64 host array -> device tensor, asynchronous when the host array is
    page-locked (stream-ordered on the current stream)."""
    h = np.ascontiguousarray(a, dtype=np.int64)
    TRAFFIC["h2d"] += h.nbytes
    return torch.from_numpy(h).to(require_cuda(), non_blocking=True)


def require_cuda() -> torch.device:
    """The current CUDA device; raises without one (no CPU fallback).  The
    availability check and the library load run once per process."""
    global _READY
    if not _READY:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_1810_06860_b200 needs a CUDA device (B200, sm_100a); it has no CPU fallback")
        _native.load()
        _READY = True
    idx = torch._C._cuda_getDevice()
    dev = _DEVICES.get(idx)
    if dev is None:
        if _DEVICES:
            # one device per process: the scratch arena, the cached device
            # patterns and the native library's per-kernel opt-ins and SM
            # count are process-wide (run one process per GPU, as torchrun does)
            raise RuntimeError(
                f"paper_1810_06860_b200 serves one CUDA device per process; already bound to "
                f"cuda:{next(iter(_DEVICES))}, now asked for cuda:{idx}")
        dev = _DEVICES[idx] = torch.device("cuda", idx)
    return dev


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    """cudaStream_t of torch's current stream on the current device (the raw
    C accessor: the Python-level current_stream() costs microseconds per
    native call)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def ld(t) -> int:
    """Row stride of a row-major (rows, cols) view."""
    if t.dim() != 2:
        raise ValueError("expected a 2-D block")
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise ValueError("expected unit column stride")
    return max(int(t.stride(0)), int(t.shape[1]), 1)


def padded_ld(cols: int) -> int:
    """Row stride (elements) of a new block: a power of two up to 8 columns,
    else a multiple of 16, so every row starts on a 128-byte line (fp64; 64
    bytes for fp32) and a gathered row of b bytes touches ceil(b / 128) lines
    -- the sparse kernels are bound by L1 wavefronts, one per line touched."""
    if cols <= 8:
        return 2 if cols <= 2 else (4 if cols <= 4 else 8)
    return (cols + 15) & ~15


def empty(rows: int, cols: int) -> torch.Tensor:
    dev = require_cuda()
    base = torch.empty((max(rows, 1), padded_ld(cols)), dtype=F64, device=dev)
    return base[:rows, :cols]


def empty32(rows: int, cols: int) -> torch.Tensor:
    """fp32 row-major block (fp32 mode), even leading dimension (8-byte
    aligned rows for the float2 SpMM path)."""
    dev = require_cuda()
    base = torch.empty((max(rows, 1), padded_ld(cols)), dtype=torch.float32, device=dev)
    return base[:rows, :cols]


def to_f32(x, out=None) -> torch.Tensor:
    """fp64 device block -> fp32 device block (lr_convert_f64_to_f32)."""
    from . import _native

    rows, cols = (int(x.shape[0]), int(x.shape[1])) if x.dim() == 2 else (1, int(x.shape[0]))
    if out is None:
        out = empty32(rows, cols) if x.dim() == 2 else torch.empty(cols, dtype=torch.float32, device=x.device)
    _native.call("lr_convert_f64_to_f32", ptr(x), ld(x) if x.dim() == 2 else cols, ptr(out),
                 ld(out) if out.dim() == 2 else cols, rows, cols, stream())
    return out


def to_f64(x, out=None) -> torch.Tensor:
    """fp32 device block -> fp64 device block (lr_convert_f32_to_f64)."""
    from . import _native

    rows, cols = int(x.shape[0]), int(x.shape[1])
    if out is None:
        out = empty(rows, cols)
    _native.call("lr_convert_f32_to_f64", ptr(x), ld(x), ptr(out), ld(out), rows, cols, stream())
    return out


def zeros(rows: int, cols: int) -> torch.Tensor:
    t = empty(rows, cols)
    if rows and cols:
        _native.call("lr_fill_f64", ptr(t), ld(t), rows, cols, 0.0, stream())
    return t


def vector(n: int) -> torch.Tensor:
    return torch.empty(max(n, 1), dtype=F64, device=require_cuda())[:n]


def to_device(x, *, copy=True) -> torch.Tensor:
    """numpy/torch 2-D float64 -> device block with unit column stride."""
    if isinstance(x, torch.Tensor):
        if x.device.type == "cuda" and x.dtype == F64 and x.dim() == 2 and (x.stride(1) == 1 or x.shape[1] <= 1):
            return x
        x = x.detach()
        if x.device.type == "cuda":
            x = x.to(F64)
            out = empty(*x.shape)
            out.copy_(x)
            return out
        x = x.numpy()
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D array, got shape {a.shape}")
    out = empty(*a.shape)
    if a.size:
        host = torch.from_numpy(np.ascontiguousarray(a))
        out.copy_(host, non_blocking=False)
        TRAFFIC["h2d"] += a.nbytes
    return out


# Device -> host copies of at least this many bytes land in page-locked
# memory from torch's caching host allocator (full-rate DMA, no staging copy);
# the returned numpy array keeps its pinned block alive and hands it back to
# the cache when it dies.
PINNED_D2H_MIN_BYTES = 1 << 20


# Small device results queued for the host in one batch (prefetch_host): the
# copies land in one page-locked buffer behind the work already queued, and the
# reads that follow (to_host of the same tensors) cost one event wait instead
# of one blocking cudaMemcpy each (rsvd_bki reads five small vectors per call).
_PREFETCHED = {}
_PREFETCH_BUF = [None]


def prefetch_host(tensors) -> None:
    """Queue device -> host copies of small contiguous tensors behind the work
    already on the stream; the next to_host() of each returns the prefetched
    values after one event wait.  The caller keeps the tensors alive, queues
    no write to them in between, and calls clear_prefetched() when done."""
    _PREFETCHED.clear()
    ts = [t.detach() for t in tensors if t is not None and not isinstance(t, np.ndarray)]
    ts = [t for t in ts if t.device.type == "cuda" and t.is_contiguous() and t.numel() > 0]
    total = sum(8 * ((int(t.numel()) * t.element_size() + 7) // 8) for t in ts)
    if not ts or total > (1 << 19):
        return
    buf = _PREFETCH_BUF[0]
    if buf is None or buf.numel() < total:
        buf = _PREFETCH_BUF[0] = torch.empty(max(2 * total, 1 << 15), dtype=torch.uint8, pin_memory=True)
    off = 0
    done = torch.cuda.Event()
    for t in ts:
        nb = int(t.numel()) * t.element_size()
        view = buf[off:off + nb].view(t.dtype)
        view.copy_(t.reshape(-1), non_blocking=True)
        _PREFETCHED[(t.data_ptr(), int(t.numel()), t.dtype)] = (view, tuple(t.shape), done)
        off += 8 * ((nb + 7) // 8)
    done.record(torch.cuda.current_stream())


def clear_prefetched() -> None:
    _PREFETCHED.clear()


def to_host(t) -> np.ndarray:
    if isinstance(t, np.ndarray):
        return t
    t = t.detach()
    if _PREFETCHED:
        hit = _PREFETCHED.pop((t.data_ptr(), int(t.numel()), t.dtype), None)
        if hit is not None and tuple(t.shape) == hit[1]:
            view, shape, done = hit
            done.synchronize()
            out = view.numpy().reshape(shape).copy()
            TRAFFIC["d2h"] += out.nbytes
            return out
    nbytes = t.numel() * t.element_size()
    if t.device.type == "cuda" and nbytes >= PINNED_D2H_MIN_BYTES:
        host = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        host.copy_(t)
        out = host.numpy()
    else:
        out = t.contiguous().cpu().numpy()
    TRAFFIC["d2h"] += out.nbytes
    return out


_SIDE = {}


def side_stream() -> torch.cuda.Stream:
    """A second stream for copies that overlap the compute stream."""
    dev = require_cuda()
    st = _SIDE.get(dev.index)
    if st is None:
        st = _SIDE[dev.index] = torch.cuda.Stream(device=dev)
    return st


class PendingHost:
    """A device->host copy in flight on the side stream (to_host_async)."""

    def __init__(self, host: torch.Tensor, done: torch.cuda.Event):
        self.host, self.done = host, done

    def result(self) -> np.ndarray:
        self.done.synchronize()
        out = self.host.numpy()
        TRAFFIC["d2h"] += out.nbytes
        return out


def to_host_async(t) -> PendingHost:
    """Start copying device tensor t into pinned host memory on the side
    stream, ordered after the work already queued on the compute stream, so
    the transfer overlaps whatever the compute stream does next."""
    t = t.detach()
    cur = torch.cuda.current_stream()
    side = side_stream()
    ready = torch.cuda.Event()
    ready.record(cur)
    host = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    with torch.cuda.stream(side):
        side.wait_event(ready)
        host.copy_(t, non_blocking=True)
        done = torch.cuda.Event()
        done.record(side)
    t.record_stream(side)  # the allocator must not recycle t before the copy ran
    return PendingHost(host, done)


def f64_upload_async(a: np.ndarray):
    """(device tensor, event): an H2D copy of host float64 data started on the
    side stream (asynchronous when a is page-locked).  The consumer waits on
    the event on its own stream before use."""
    h = np.ascontiguousarray(a, dtype=np.float64)
    TRAFFIC["h2d"] += h.nbytes
    dev = require_cuda()
    side = side_stream()
    out = torch.empty(h.shape, dtype=torch.float64, device=dev)
    with torch.cuda.stream(side):
        out.copy_(torch.from_numpy(h), non_blocking=True)
        done = torch.cuda.Event()
        done.record(side)
    out.record_stream(side)
    return out, done


_NP_TO_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
                np.dtype(np.int32): torch.int32, np.dtype(np.uint8): torch.uint8}


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A page-locked copy of a host array (numpy view of a pinned torch
    buffer): host -> device uploads from it are direct DMA transfers."""
    a = np.ascontiguousarray(a)
    t = torch.empty(a.shape, dtype=_NP_TO_TORCH[a.dtype], pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out


SMALL_ASYNC_BYTES = 1 << 20  # small uploads go through pinned staging, without a stream sync


def _upload(h: np.ndarray, dtype) -> torch.Tensor:
    """Host array -> device.  Small arrays (the S vectors, column lists of a
    call) are staged in pinned memory and copied without blocking, so the
    upload does not synchronise the stream (a pageable .to(cuda) does); the
    caching host allocator keeps the staging block until the copy ran."""
    TRAFFIC["h2d"] += h.nbytes
    dev = require_cuda()
    if h.nbytes <= SMALL_ASYNC_BYTES:
        st = torch.empty(h.shape, dtype=dtype, pin_memory=True)
        st.numpy()[...] = h
        return st.to(dev, non_blocking=True)
    return torch.from_numpy(h).to(dev)


def int_buffer(a: np.ndarray) -> torch.Tensor:
    return _upload(np.ascontiguousarray(a, dtype=np.int32), torch.int32)


def f64_buffer(a: np.ndarray) -> torch.Tensor:
    return _upload(np.ascontiguousarray(a, dtype=np.float64), torch.float64)


class Arena:
    """Named, grow-only scratch buffers (float64) reused across calls."""

    def __init__(self):
        self._bufs = {}

    def get(self, name: str, ndoubles: int) -> torch.Tensor:
        n = max(int(ndoubles), 1)
        b = self._bufs.get(name)
        if b is None or b.numel() < n:
            b = torch.empty(int(n * 1.25) + 64, dtype=F64, device=require_cuda())
            self._bufs[name] = b
        return b


_ARENA = None


def arena() -> Arena:
    global _ARENA
    if _ARENA is None:
        _ARENA = Arena()
    return _ARENA
