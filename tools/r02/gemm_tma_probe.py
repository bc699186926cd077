"""TMA / mbarrier GEMM mainloop (LR_GEMM_TILE=6) against the cp.async kernels
on the BKI / SVT shapes: correctness against torch (cuBLAS) and time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1810_06860_b200 import device, linalg
rng = np.random.default_rng(0)
cases = []
for m, W, k in ((100000, 660, 100), (138493, 220, 50), (138493, 110, 50)):
    H = device.to_device(rng.standard_normal((m, W)))
    R = device.to_device(np.triu(rng.standard_normal((W, W))))
    V = device.to_device(rng.standard_normal((W, k)))
    Ht = H.clone()
    cases += [(f"syrk {m}x{W}", lambda H=H: linalg.gram_dev(H), m * W * (W + 1), lambda H=H: H.T @ H),
              (f"nn_upper {m}x{W}x{W}", lambda H=H, R=R: linalg.matmul_dev(H, R, b_upper=True), m * W * (W + 1),
               lambda H=H, R=R: H @ R),
              (f"nn {m}x{W}x{k}", lambda H=H, V=V: linalg.matmul_dev(H, V), 2 * m * W * k, lambda H=H, V=V: H @ V),
              (f"tn {m}x{W}x{W}", lambda H=H, Ht=Ht: linalg.matmul_tn_dev(H, Ht), 2 * m * W * W,
               lambda H=H, Ht=Ht: H.T @ Ht)]
tag = os.environ.get("LR_GEMM_TILE", "default")
for name, fn, flops, ref in cases:
    got = fn()
    r = ref()
    err = float(torch.linalg.norm(got - r) / torch.linalg.norm(r))
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    print(f"tile={tag} {name:26s} {ms:.3f} ms  {flops / ms / 1e9:6.2f} TFLOP/s  rel err vs cuBLAS {err:.1e}", flush=True)
