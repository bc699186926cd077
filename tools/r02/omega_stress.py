"""Stress of the device-assembled Omega path: cfg4 jobs with the staging slots dropped before each job (so the
slot buffers are reallocated and grown inside every job, as in a process's first job); every job must reproduce
the reference trace (71 iterations, the golden residual)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_1810_06860_b200 import completion, rng, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o4 = workloads.cfg4()
obs = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
params = bench.cfg4_params()
eng = completion.DeviceEngine(obs)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad = 0
ref_tr = None
for rep in range(n):
    if os.environ.get("STRESS_KEEP_STATE") != "1":  # default: every job starts like a process's first job
        rng._STAGING.clear(); rng._STAGING_NEXT[0] = 0; rng._SUPERSETS.clear(); rng._PREFETCH.clear()
        torch.cuda.empty_cache()
    try:
        res = completion._svt_loop(obs, params, "rsvd-bki", params.strategy, engine=eng)
        ok = res.iterations == 71 and abs(res.residual - 0.39918764231064247) < 1e-9
        tr = [(t.k, t.r, t.p, t.q, t.svd_source, t.residual) for t in res.trace]
        if rep == 0 and ok:
            ref_tr = tr
        note = ""
        if not ok and ref_tr is not None:
            for a, b in zip(ref_tr, tr):
                if a[:5] != b[:5] or abs(a[5] - b[5]) > 1e-13 * abs(a[5]):
                    note = f" first deviation at iteration {ref_tr.index(a) + 1}: ref {a} got {b}"
                    break
        print(rep, res.iterations, res.residual, "ok" if ok else "MISMATCH" + note, flush=True)
    except Exception as exc:  # noqa: BLE001
        ok = False
        print(rep, "ERROR", type(exc).__name__, str(exc)[:120], flush=True)
    bad += not ok
print("bad", bad, "of", n)
