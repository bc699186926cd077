"""Is one rsvd_bki call deterministic?  The same call (cfg4 train matrix, k = 15 / 27, p = 2) repeated with the
device Omega (no host draw involved) and with the host Omega; singular values compared bit for bit."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1810_06860_b200 import rsvd, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o4 = workloads.cfg4()
A = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split).train_matrix()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
import os
from paper_1810_06860_b200 import device
if os.environ.get("NO_PREFETCH") == "1":  # the five reads of a call as separate blocking copies
    device.prefetch_host = lambda tensors: None
if os.environ.get("FILL"):  # every fresh block / vector / arena buffer pre-filled: do uninitialised recycled buffers leak into the result?
    fillv = float(os.environ["FILL"])
    _empty, _vector = device.empty, device.vector
    def _e(rows, cols):
        t = _empty(rows, cols); t._base.fill_(fillv) if t._base is not None else t.fill_(fillv); return t
    def _v(n_):
        t = _vector(n_); t.fill_(fillv); return t
    device.empty, device.vector = _e, _v
    import paper_1810_06860_b200.linalg as _l, paper_1810_06860_b200.sparse as _s
if os.environ.get("NO_REUSE") == "1":
    rsvd.KRYLOV_REUSE = False
if os.environ.get("NO_SPEC") == "1":
    rsvd.SPECULATIVE = False
for omega in ("device",):
    for k, p in ((27, 2), (43, 3)):
        prm = rsvd.RsvdParams(k=k, p=p, s=5, seed=1234 + k)
        ref = None
        bad = []
        t0 = time.perf_counter()
        for rep in range(n):
            res, _, _ = rsvd.rsvd_bki_dev(A, prm, allow_fallback=True, omega=omega)
            S = res.S_host.copy()
            if ref is None:
                ref = S
            elif not np.array_equal(S, ref):
                bad.append((rep, float(np.max(np.abs(S - ref) / ref))))
        print(f"omega={omega} k={k} p={p}: {n} calls in {time.perf_counter() - t0:.1f} s, deviating {len(bad)} {bad[:5]}", flush=True)
