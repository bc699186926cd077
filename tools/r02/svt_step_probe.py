"""Fused SVT step (lr_svt_step_f64, apply = 1) on the cfg4 train pattern at
fixed ranks: device time per launch (CUDA events, median of 7 after 3 warm),
compulsory HBM bytes and the V-gather rate.  RANKS=10,48,84 by default.
NCU=1: run each rank exactly twice (one warm + one captured) for ncu."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1810_06860_b200 import workloads, device, completion, profiling
from paper_1810_06860_b200.sparse import ObservationSet

o = workloads.cfg4()
eng = completion.DeviceEngine(ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split))
eng.m_norm = eng.observed_norm()
eng.start(1.0)
m, n, nnz = eng.m, eng.n, eng.nnz
rng = np.random.default_rng(0)
ncu = os.environ.get("NCU") is not None
completion.CSC_SCATTER = os.environ.get("SCATTER") == "1"
from paper_1810_06860_b200 import sparse as _sp
if os.environ.get("LR_SVT_KERNEL"):
    _sp.SVT_KERNEL = "items"
tag = (f"[family={_sp.SVT_KERNEL} kernel={os.environ.get('LR_SVT_KERNEL', '-')} "
       f"gt={os.environ.get('LR_SVT_FLAT', os.environ.get('LR_SVT_GT', 'auto'))} scatter={int(completion.CSC_SCATTER)}]")
for r in [int(x) for x in os.environ.get("RANKS", "10,48,84").split(",")]:
    U = device.to_device(rng.standard_normal((m, r)) * 0.01)
    V = device.to_device(rng.standard_normal((n, r)) * 0.01)
    S = rng.random(r) + 1.0
    ts, tg = [], []
    for it in range(2 if ncu else 10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        resid, _ = eng.step(U, S, V, r, 1e-9)
        e1.record()
        eng.Y.device_values()  # CSC refresh (no-op with the in-step scatter)
        e2.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); tg.append(e1.elapsed_time(e2))
    ms = float(np.median(ts[3:] if not ncu else ts))
    mg = float(np.median(tg[3:] if not ncu else tg))
    b40 = 4 * (m + 1) + 40 * nnz + 8 * (m + n) * r + 8 * r
    b28 = b40 - 12 * nnz
    print(f"{tag} r={r}: step {ms*1e3:.1f} us (incl. finish + residual D2H), csc refresh {mg*1e3:.1f} us | "
          f"40B model {b40/ms/1e6:.0f} GB/s = {b40/ms/1e6/6547.5:.3f} of HBM | 28B model {b28/ms/1e6:.0f} GB/s "
          f"| step+refresh on 40B {b40/(ms+mg)/1e6/6547.5:.3f} | V gather {nnz*8*r/ms/1e9:.2f} TB/s", flush=True)
