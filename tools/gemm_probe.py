# Time the BKI-shaped dense products (median of 10) with algorithmic TFLOP/s.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
rng = np.random.default_rng(0)
H = device.to_device(rng.standard_normal((100000, 660)))
Bt = device.to_device(rng.standard_normal((50000, 660)))
R = device.to_device(np.triu(rng.standard_normal((660, 660))))
V = device.to_device(rng.standard_normal((660, 100)))
cases = (("syrk 100000x660", lambda: linalg.gram_dev(H), 100000 * 660 * 661),
         ("syrk 50000x660", lambda: linalg.gram_dev(Bt), 50000 * 660 * 661),
         ("nn_upper 100000x660x660", lambda: linalg.matmul_dev(H, R, b_upper=True), 100000 * 660 * 661),
         ("nn 100000x660x100", lambda: linalg.matmul_dev(H, V), 2 * 100000 * 660 * 100),
         ("nn 50000x660x100", lambda: linalg.matmul_dev(Bt, V), 2 * 50000 * 660 * 100))
for name, fn, flops in cases:
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    print(f"{name:26s} {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s (algorithmic)", flush=True)
