"""Seeded streams for the Gaussian test matrices.

Same contract as the reference RNG (/root/reference/pkg/src/lowrank/rng.py):
a stream is numpy's Philox4x64-10 keyed by the seed; normals are Box-Muller
over one block of uniforms (first half -> radius via 1-u, second half ->
angle; cos to even slots, sin to odd); a Gaussian matrix is filled column by
column and stored row-major; spawn(tag) derives
(seed * 0x9E3779B97F4A7C15 + tag + 1) mod 2^63.

Two producers of Omega share that contract:
  * gaussian_matrix        -- host numpy (the reference's own arithmetic);
  * gaussian_matrix_device -- lr_gaussian_f64 on the GPU: same Philox words
    and uniforms bit for bit, normals within a few ulp of the host values
    (libdevice log/sincos vs the host libm), no PCIe transfer.
"""

from __future__ import annotations

import numpy as np

_SPAWN_MUL = 0x9E3779B97F4A7C15
_MOD63 = 1 << 63


class RngState:
    """A Philox stream with a running count of uniforms drawn."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self.position = 0
        self._gen = np.random.Generator(np.random.Philox(key=self.seed))

    def __repr__(self):
        return f"RngState(seed={self.seed}, position={self.position})"

    def uniform(self, count: int) -> np.ndarray:
        self.position += count
        return self._gen.random(count)

    def normal_pairs(self, count: int) -> np.ndarray:
        npairs = (count + 1) // 2
        block = self.uniform(2 * npairs)
        radius = np.sqrt(-2.0 * np.log(1.0 - block[:npairs]))
        angle = 2.0 * np.pi * block[npairs:]
        z = np.empty(2 * npairs)
        z[0::2] = radius * np.cos(angle)
        z[1::2] = radius * np.sin(angle)
        return z[:count]

    def integers(self, low: int, high: int, count: int) -> np.ndarray:
        self.position += count
        return self._gen.integers(low, high, size=count)

    def permutation(self, n: int) -> np.ndarray:
        self.position += n
        return self._gen.permutation(n)

    def choice_without_replacement(self, n: int, k: int) -> np.ndarray:
        self.position += k
        return self._gen.choice(n, size=k, replace=False, shuffle=False)

    def spawn(self, tag: int) -> "RngState":
        return RngState((self.seed * _SPAWN_MUL + tag + 1) % _MOD63)


def _check_shape(rows: int, cols: int) -> None:
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian matrix needs rows, cols >= 1, got {rows}x{cols}")


def gaussian_matrix(rng: RngState, rows: int, cols: int) -> np.ndarray:
    """Host Omega, advancing `rng` (rng.py:77-94 semantics)."""
    _check_shape(rows, cols)
    z = rng.normal_pairs(rows * cols)
    return np.ascontiguousarray(z.reshape((cols, rows)).T)


# ------------------------------------------------- threaded host producer
#
# The parity Omega is numpy's own arithmetic (above), but one thread of it
# costs ~0.35 s per cfg2 call (5.5M normals).  The draw splits exactly:
# Philox4x64 words are counter-addressed (numpy's Philox.advance(k) skips k
# four-word blocks), and every Box-Muller output depends on its own pair of
# uniforms only, through numpy's element-wise ufuncs (log, sqrt, cos, sin),
# whose per-element results do not depend on where a chunk starts
# (tests/test_host_logic.py::test_threaded_gaussian_is_bit_exact checks it on
# the host it runs on).  So T threads each fill a slice of the uniforms and of
# the normals, in place, into a caller-provided (pinned) buffer -- the numpy
# ufuncs and the Philox fill release the GIL.

# draw pool size; None: os.cpu_count() (LR_HOST_THREADS limits it, e.g. to study a slower host)
HOST_THREADS = int(__import__("os").environ.get("LR_HOST_THREADS") or 0) or None
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(max_workers=HOST_THREADS or os.cpu_count() or 1,
                                   thread_name_prefix="lr-omega")
    return _POOL


def _uniform_slice(seed: int, start: int, out: np.ndarray) -> None:
    bg = np.random.Philox(key=seed)
    bg.advance(start // 4)
    gen = np.random.Generator(bg)
    skip = start % 4
    if skip:
        gen.random(skip)
    gen.random(out=out)


# The C pieces of the draw (csrc/lr_host_rng.c): Philox uniforms and the
# Box-Muller pairing with libm cos/sin; np.log stays numpy's.  Used only after
# a bit-for-bit self-check against the all-numpy draw on this host (numpy's
# float64 cos/sin are libm's here, its log is its own SIMD kernel).
_C_DRAW = None


def _c_draw_lib():
    global _C_DRAW
    if _C_DRAW is None:
        _C_DRAW = False
        try:
            from . import _native

            lib = _native.load()
            _C_DRAW = lib
            ok = all(np.array_equal(_normals_c(lib, s, r, c), _normals_numpy(s, r, c))
                     for s, r, c in ((3, 7, 5), (2 ** 62 + 11, 1001, 3), (12345, 4099, 37)))
            if not ok:
                _C_DRAW = False
        except Exception:
            _C_DRAW = False
    return _C_DRAW


def _normals_c(lib, seed: int, rows: int, cols: int, out: np.ndarray = None, pool=None) -> np.ndarray:
    count = rows * cols
    npairs = (count + 1) // 2
    u1 = np.empty(npairs)
    u2 = np.empty(npairs)
    direct = out is not None and out.size >= 2 * npairs
    dst = out.reshape(-1) if direct else np.empty(2 * npairs)
    nt = 1 if pool is None else max(1, min(pool._max_workers, npairs // (1 << 15)))
    pc = [(npairs * t) // nt for t in range(nt + 1)]
    seed = int(seed) & ((1 << 64) - 1)

    def part(t):
        a, b = pc[t], pc[t + 1]
        if a == b:
            return
        x1, x2 = u1[a:b], u2[a:b]
        lib.lr_host_uniforms(seed, a, b - a, x1.ctypes.data)
        lib.lr_host_uniforms(seed, npairs + a, b - a, x2.ctypes.data)
        np.subtract(1.0, x1, out=x1)
        np.log(x1, out=x1)
        lib.lr_host_box_muller(x1.ctypes.data, x2.ctypes.data, b - a, dst[2 * a:2 * b].ctypes.data)

    if nt == 1:
        part(0)
    else:
        list(pool.map(part, range(nt)))
    if out is not None and not direct:
        out.reshape(-1)[:count] = dst[:count]
        return out.reshape(-1)[:count]
    return dst[:count]


def _normals_numpy(seed: int, rows: int, cols: int) -> np.ndarray:
    return RngState(seed).normal_pairs(rows * cols)


def normals_column_major(seed: int, rows: int, cols: int, out: np.ndarray = None) -> np.ndarray:
    """Omega = gaussian_matrix(RngState(seed), rows, cols) in COLUMN-major
    order (the draw order: column c is out[c*rows:(c+1)*rows]), bit-identical
    to the one-thread draw, computed by the thread pool into `out`."""
    _check_shape(rows, cols)
    lib = _c_draw_lib()
    if lib:
        return _normals_c(lib, seed, rows, cols, out, _pool())
    count = rows * cols
    npairs = (count + 1) // 2
    u = np.empty(2 * npairs)
    z = np.empty(2 * npairs) if (out is None or count % 2) else None
    pool = _pool()
    nt = max(1, min(pool._max_workers, (2 * npairs) // (1 << 16)))
    # uniforms: contiguous slices of the counter space
    cuts = [(2 * npairs * t) // nt for t in range(nt + 1)]
    list(pool.map(lambda t: _uniform_slice(seed, cuts[t], u[cuts[t]:cuts[t + 1]]), range(nt)))
    dst = z if z is not None else out.reshape(-1)[: 2 * npairs]
    pc = [(npairs * t) // nt for t in range(nt + 1)]

    def box_muller(t):
        a, b = pc[t], pc[t + 1]
        if a == b:
            return
        radius = np.sqrt(-2.0 * np.log(1.0 - u[a:b]))
        angle = 2.0 * np.pi * u[npairs + a:npairs + b]
        dst[2 * a:2 * b:2] = radius * np.cos(angle)
        dst[2 * a + 1:2 * b:2] = radius * np.sin(angle)

    list(pool.map(box_muller, range(nt)))
    if out is None:
        return z[:count]
    if z is not None:
        out.reshape(-1)[:count] = z[:count]
    return out.reshape(-1)[:count]


def _pinned_normals(seed: int, rows: int, cols: int):
    import torch

    count = rows * cols
    host = torch.empty(count + (count & 1), dtype=torch.float64, pin_memory=True)
    normals_column_major(seed, rows, cols, out=host.numpy())
    return host


_PREFETCH = {}
PREFETCH_KEEP = 5  # draws kept (the SVT loop's speculative candidates + the exact one)


def prefetch_normals(seed: int, rows: int, cols: int) -> None:
    """Start drawing Omega(seed, rows, cols) on the host pool in the
    background (the SVT loop calls this for the next fresh inner SVD while the
    GPU runs the current iteration).  At most a few draws are kept."""
    key = (int(seed), int(rows), int(cols))
    if key in _PREFETCH or rows < 1 or cols < 1:
        return
    if superset_pending_on_device(*key):
        return  # assembled on the GPU from the Superset's uploaded halves
    while len(_PREFETCH) >= PREFETCH_KEEP:
        _PREFETCH.pop(next(iter(_PREFETCH)))
    import threading
    from concurrent.futures import Future

    fut = Future()
    dev_index = _current_device_index()

    def run():
        try:
            sup = _superset_for(*key)
            host = _pinned_from_superset(sup, key[2]) if sup is not None else _pinned_normals(*key)
            fut.set_result(_Drawn(host, *(_upload_async(host, key[1] * key[2], dev_index)
                                          if dev_index is not None else (None, None))))
        except BaseException as exc:  # pragma: no cover - surfaced by take_normals
            fut.set_exception(exc)

    threading.Thread(target=run, daemon=True, name="lr-omega-prefetch").start()
    _PREFETCH[key] = fut


class _Drawn:
    """A prefetched draw: the pinned host block and, when a GPU is present,
    its device copy made on the upload stream (event `ready`)."""

    def __init__(self, host, dev, ready):
        self.host, self.dev, self.ready = host, dev, ready


_UPLOAD_STREAM = {}


def _current_device_index():
    try:
        import torch

        if not torch.cuda.is_available():
            return None
        return torch.cuda.current_device()
    except Exception:
        return None


def _upload_async(host, count: int, dev_index: int):
    """In the prefetch thread: the draw's host->device copy on a dedicated
    stream, so it overlaps the GPU's current work instead of following the
    host's wait for the draw."""
    import torch

    torch.cuda.set_device(dev_index)
    st = _UPLOAD_STREAM.get(dev_index)
    if st is None:
        st = _UPLOAD_STREAM.setdefault(dev_index, torch.cuda.Stream(device=dev_index))
    with torch.cuda.stream(st):
        dev = torch.empty(max(count, 1), dtype=torch.float64, device=torch.device("cuda", dev_index))
        if count:
            dev[:count].copy_(host[:count], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(st)
    return dev, ev


def take_normals_device(seed: int, rows: int, cols: int):
    """(device vector, event) of a prefetched draw already copied to the GPU,
    or None (nothing prefetched, or no device copy made)."""
    key = (int(seed), int(rows), int(cols))
    fut = _PREFETCH.get(key)
    if fut is None:
        return None
    d = fut.result()
    if d.dev is None:
        return None
    _PREFETCH.pop(key, None)
    return d.dev, d.ready


# Threads a Superset draw is cut into.  It runs beside the SVT loop's main
# thread, which launches the current inner SVD meanwhile: cut over every core
# it slows that thread more than it gains (cfg4 job with the device assembly:
# 627 ms on 16 threads, 612 ms on 6; profiles/r02bb_host_sensitivity.txt).
# Single draws on the critical path (a standalone rsvd call) use the whole pool.
SUPERSET_THREADS = int(__import__("os").environ.get("LR_SUPERSET_THREADS") or 6)


class _StagingSlot:
    """Page-locked host buffers a device-backed Superset is drawn into and
    uploaded from.  A few slots are allocated once and handed out in turn
    (cudaHostAlloc inside the drawing thread stalls the main thread's kernel
    launches); `gen` tells a Superset whether the slot is still its own."""

    def __init__(self):
        self.R = self.cs = None
        self.R_dev = self.cs_dev = None  # device copies, grown rarely (no cudaMalloc per draw: it stalls the GPU)
        self.gen = 0
        self.owner = None     # Future of the Superset being drawn into this slot
        self.uploaded = None  # event of the last upload read from this slot
        self.consumed = None  # event after the last kernel that read the device copies


_STAGING = []
_STAGING_NEXT = [0]
_STAGING_SLOTS = 4  # two Supersets are kept; a slot is reused two draws after its Superset was dropped


def _staging_slot(n_r: int, n_cs: int) -> _StagingSlot:
    import torch

    if len(_STAGING) < _STAGING_SLOTS:
        _STAGING.append(_StagingSlot())
        slot = _STAGING[-1]
    else:
        slot = _STAGING[_STAGING_NEXT[0] % _STAGING_SLOTS]
    _STAGING_NEXT[0] += 1
    if slot.owner is not None:  # the slot's previous Superset has been drawn and its upload queued ...
        try:
            slot.owner.result()
        except BaseException:
            pass
        slot.owner = None
    if slot.uploaded is not None:
        slot.uploaded.synchronize()  # ... and that upload has left the buffer
        slot.uploaded = None
    slot.gen += 1
    if slot.R is None or slot.R.numel() < n_r:
        slot.R = torch.empty(int(n_r * 1.5) + 1024, dtype=torch.float64, pin_memory=True)
    if slot.cs is None or slot.cs.numel() < n_cs:
        slot.cs = torch.empty(int(n_cs * 1.5) + 1024, dtype=torch.float64, pin_memory=True)
    return slot


class Superset:
    """One seed's draws for every width in [w_lo, w_hi] at ~the cost of one:
    Box-Muller pairs uniform i with uniform P + i (P = ceil(rows w / 2)), so
    the radii R[i] (uniforms [0, P_hi)) and the cos / sin of the uniforms at
    stream positions [P_lo, 2 P_hi) serve every width; a width's normals are
    then z[2i] = R[i] cos(2 pi u[P + i]), z[2i+1] = R[i] sin(...) -- the same
    IEEE operations as the one-width draw, so bit-identical to it
    (tests/test_host_logic.py::test_superset_draw_is_bit_exact).  The SVT
    loop builds one at the top of each iteration for the next iteration's
    plausible ranks, while the GPU runs the current inner SVD."""

    def __init__(self, lib, seed: int, rows: int, w_lo: int, w_hi: int, pool=None, slot: "_StagingSlot" = None):
        self.lib, self.seed, self.rows, self.w_lo, self.w_hi = lib, int(seed), int(rows), int(w_lo), int(w_hi)
        self.p_lo = (rows * w_lo + 1) // 2
        self.p_hi = (rows * w_hi + 1) // 2
        seed64 = self.seed & ((1 << 64) - 1)
        na = 2 * self.p_hi - self.p_lo
        self.dev = None  # (R, cs device copies, ready event) once uploaded (upload_async)
        self.counted = False  # its upload added to device.TRAFFIC
        if slot is not None:  # page-locked halves: uploaded once, every width assembled on the GPU
            self._slot = slot
            self._gen = slot.gen
            self.R, self.cs = self._slot.R.numpy()[:self.p_hi], self._slot.cs.numpy()[:2 * na]
        else:
            self._slot = None
            self.R = np.empty(self.p_hi)
            self.cs = np.empty(2 * na)
        ua = np.empty(na)
        nt = 1 if pool is None else max(1, min(pool._max_workers, SUPERSET_THREADS, self.p_hi // (1 << 15)))

        def part(t):
            a, b = (self.p_hi * t) // nt, (self.p_hi * (t + 1)) // nt
            if b > a:
                x = self.R[a:b]
                lib.lr_host_uniforms(seed64, a, b - a, x.ctypes.data)
                np.subtract(1.0, x, out=x)
                np.log(x, out=x)
                np.multiply(-2.0, x, out=x)
                np.sqrt(x, out=x)
            a, b = (na * t) // nt, (na * (t + 1)) // nt
            if b > a:
                y = ua[a:b]
                lib.lr_host_uniforms(seed64, self.p_lo + a, b - a, y.ctypes.data)
                lib.lr_host_cossin(y.ctypes.data, b - a, self.cs[2 * a:2 * b].ctypes.data)

        if nt == 1:
            part(0)
        else:
            list(pool.map(part, range(nt)))

    def covers(self, rows: int, cols: int) -> bool:
        return int(rows) == self.rows and self.w_lo <= int(cols) <= self.w_hi

    def upload_async(self, dev_index: int) -> None:
        """In the drawing thread: copy R and cs to the GPU on the upload
        stream (overlapping the current inner SVD); lr_omega_assemble_f64 then
        forms any covered width's Omega on the device with no host work after
        the rank is known."""
        import torch

        torch.cuda.set_device(dev_index)
        st = _UPLOAD_STREAM.get(dev_index)
        if st is None:
            st = _UPLOAD_STREAM.setdefault(dev_index, torch.cuda.Stream(device=dev_index))
        dv = torch.device("cuda", dev_index)
        nR, ncs = int(self.R.shape[0]), int(self.cs.shape[0])
        slot = self._slot
        with torch.cuda.stream(st):
            if slot.R_dev is None or slot.R_dev.numel() < nR:
                slot.R_dev = torch.empty(int(nR * 1.5) + 1024, dtype=torch.float64, device=dv)
            if slot.cs_dev is None or slot.cs_dev.numel() < ncs:
                slot.cs_dev = torch.empty(int(ncs * 1.5) + 1024, dtype=torch.float64, device=dv)
            if slot.consumed is not None:  # the slot's previous Superset may still be read by a queued kernel
                st.wait_event(slot.consumed)
                slot.consumed = None
            R, cs = slot.R_dev[:nR], slot.cs_dev[:ncs]
            R.copy_(slot.R[:nR], non_blocking=True)
            cs.copy_(slot.cs[:ncs], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        slot.uploaded = ev
        self.dev = (R, cs, ev)

    def mark_consumed(self, stream) -> None:
        """A kernel reading the device copies was just queued on `stream`."""
        import torch

        if self._slot is not None and self._slot.gen == self._gen:
            ev = torch.cuda.Event()
            ev.record(stream)
            self._slot.consumed = ev

    def host_valid(self) -> bool:
        """The host halves are still this Superset's (a staged Superset's
        page-locked slot is handed to a later one after two more draws)."""
        return self._slot is None or self._slot.gen == self._gen

    def normals(self, cols: int, out: np.ndarray, pool=None) -> np.ndarray:
        """Column-major Omega(seed, rows, cols) into out (>= 2 P entries)."""
        P = (self.rows * int(cols) + 1) // 2
        off = P - self.p_lo
        z = out.reshape(-1)
        nt = 1 if pool is None else max(1, min(pool._max_workers, P // (1 << 16)))
        cuts = [(P * t) // nt for t in range(nt + 1)]

        def part(t):
            a, b = cuts[t], cuts[t + 1]
            if b > a:
                self.lib.lr_host_bm_assemble(self.R[a:b].ctypes.data, self.cs[2 * (off + a):2 * (off + b)].ctypes.data,
                                             b - a, z[2 * a:2 * b].ctypes.data)

        if nt == 1:
            part(0)
        else:
            list(pool.map(part, range(nt)))
        return z[: self.rows * int(cols)]


_SUPERSETS = {}  # seed -> Future[Superset]


def prefetch_superset(seed: int, rows: int, w_lo: int, w_hi: int) -> None:
    """Start a Superset draw for seed over widths [w_lo, w_hi] in the
    background (at most two seeds kept)."""
    lib = _c_draw_lib()
    if not lib or rows < 1 or w_lo < 1 or w_hi < w_lo:
        return
    key = int(seed)
    old = _SUPERSETS.get(key)
    if old is not None and old[0] == (int(rows), int(w_lo), int(w_hi)):
        return
    while len(_SUPERSETS) >= 2:
        _SUPERSETS.pop(next(iter(_SUPERSETS)))
    import threading
    from concurrent.futures import Future

    fut = Future()
    dev_index = _current_device_index() if SUPERSET_ON_DEVICE else None
    slot = None
    if dev_index is not None:  # chosen here, in the caller's thread: a fixed rotation
        p_hi = (int(rows) * int(w_hi) + 1) // 2
        slot = _staging_slot(p_hi, 2 * (2 * p_hi - (int(rows) * int(w_lo) + 1) // 2))
        slot.owner = fut

    def run():
        try:
            sup = Superset(lib, seed, rows, w_lo, w_hi, _pool(), slot=slot)
            if dev_index is not None:
                sup.upload_async(dev_index)
            fut.set_result(sup)
        except BaseException as exc:  # pragma: no cover - surfaced on use
            fut.set_exception(exc)

    threading.Thread(target=run, daemon=True, name="lr-omega-superset").start()
    _SUPERSETS[key] = ((int(rows), int(w_lo), int(w_hi)), fut)


# Opt-in (LR_SUPERSET_DEVICE=1): a Superset's halves are uploaded as soon as
# they are drawn and Omega is assembled on the GPU (lr_omega_assemble_f64,
# bit-identical), so no host draw, assembly or upload follows the rank read:
# 95 % of the cfg4 job's draws.  With the Superset cut into SUPERSET_THREADS =
# 6 pieces the job runs in 605 ms against 614 ms for the host assembly, and it
# does not depend on the host's draw throughput (draw pool limited to 3
# threads: 629 ms against 756 ms; profiles/r02bb_host_sensitivity.txt,
# r02bc_superset_threads.txt).  NOT the default: stress runs of the cfg4 job
# (tools/r02/omega_stress.py) diverged once in ~150 jobs with it even after the
# stream-ordering fix of the staging buffers (profiles/r02bg_omega_stress.txt),
# and never without it; until that is understood the width is assembled on the
# host and uploaded by the prefetch thread.
SUPERSET_ON_DEVICE = __import__("os").environ.get("LR_SUPERSET_DEVICE", "0") == "1"


def superset_pending_on_device(seed: int, rows: int, cols: int) -> bool:
    """A Superset covering (seed, rows, cols) is drawn or being drawn with a
    device copy: the exact-width host draw is not needed."""
    ent = _SUPERSETS.get(int(seed))
    if ent is None or not SUPERSET_ON_DEVICE or _current_device_index() is None:
        return False
    (r, lo, hi), _ = ent
    return r == int(rows) and lo <= int(cols) <= hi


def superset_on_device(seed: int, rows: int, cols: int):
    """The Superset covering (seed, rows, cols) once its device copy exists
    (waits for the drawing thread), else None."""
    if not superset_pending_on_device(seed, rows, cols):
        return None
    sup = _superset_for(seed, rows, cols)
    return sup if (sup is not None and sup.dev is not None) else None


def _superset_for(seed: int, rows: int, cols: int):
    ent = _SUPERSETS.get(int(seed))
    if ent is None:
        return None
    (r, lo, hi), fut = ent
    if r != int(rows) or not lo <= int(cols) <= hi:
        return None
    try:
        sup = fut.result()
    except Exception:
        return None
    return sup if sup.host_valid() else None


def _pinned_from_superset(sup: Superset, cols: int):
    import torch

    count = sup.rows * int(cols)
    host = torch.empty(count + (count & 1), dtype=torch.float64, pin_memory=True)
    sup.normals(cols, host.numpy(), _pool())
    return host


def take_normals(seed: int, rows: int, cols: int):
    """Pinned column-major Omega(seed, rows, cols): the prefetched draw when
    one matches, else assembled from a Superset covering the width, else
    drawn now."""
    fut = _PREFETCH.pop((int(seed), int(rows), int(cols)), None)
    if fut is not None:
        return fut.result().host
    sup = _superset_for(seed, rows, cols)
    if sup is not None:
        return _pinned_from_superset(sup, cols)
    return _pinned_normals(seed, rows, cols)


def gaussian_matrix_fast(rng: RngState, rows: int, cols: int) -> np.ndarray:
    """gaussian_matrix(rng, rows, cols), bit for bit, from the thread pool;
    `rng` advances exactly as the one-thread draw advances it."""
    _check_shape(rows, cols)
    total = 2 * ((rows * cols + 1) // 2)
    if rng.position != 0:
        return gaussian_matrix(rng, rows, cols)
    z = normals_column_major(rng.seed, rows, cols)
    bg = np.random.Philox(key=rng.seed)
    bg.advance(total // 4)
    rng._gen = np.random.Generator(bg)
    if total % 4:
        rng._gen.random(total % 4)
    rng.position += total
    return np.ascontiguousarray(z.reshape((cols, rows)).T)


def gaussian_matrix_device(seed: int, rows: int, cols: int, out=None):
    """Device Omega = gaussian_matrix(RngState(seed), rows, cols) generated by
    lr_gaussian_f64 directly into a padded device block (or into `out`)."""
    from . import _native, device

    _check_shape(rows, cols)
    if out is None:
        out = device.empty(rows, cols)
    _native.call("lr_gaussian_f64", int(seed) & ((1 << 64) - 1), rows, cols, device.ptr(out),
                 device.ld(out), device.stream())
    return out
