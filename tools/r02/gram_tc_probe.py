"""tcgen05 3xTF32 Gram (fp32 mode) against the fp64 DMMA Gram at the eigSVD
shapes of cfg2 (n = 50000 / m = 100000 rows, W = 110 / 660) and cfg4
(26744 rows, W = 100..300): CUDA-event time per call (L2 flushed between
calls), algorithmic bytes (K n 4 for fp32, K n 8 for fp64) and the accuracy
against the fp64 Gram."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_06860_b200 import device, linalg  # noqa: E402

flush = torch.empty(64 * 2**20, dtype=torch.float64, device="cuda")


def timed(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()  # the native calls run on torch's current stream
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e-3


for K, n in ((50000, 110), (50000, 660), (100000, 660), (26744, 100), (26744, 300), (138493, 300)):
    A = torch.randn(K, n, dtype=torch.float64, device="cuda")
    A64 = device.empty(K, n)
    A64.copy_(A)
    A32 = device.to_f32(A64)
    t32 = timed(lambda: linalg.gram_tf32x3_dev(A32))
    t64 = timed(lambda: linalg.gram_dev(A64))
    G32 = linalg.gram_tf32x3_dev(A32)
    A3 = device.to_f64(A32)
    G64 = linalg.gram_dev(A3)
    d = torch.sqrt(torch.diagonal(G64))
    err = float(torch.max(torch.abs(G32 - G64) / torch.outer(d, d)))
    print(f"K={K:7d} n={n:4d}: tf32x3 {t32 * 1e6:8.1f} us ({K * n * 4 / t32 / 1e9:7.0f} GB/s, "
          f"{K * n * n * 3 / t32 / 1e12:6.1f} TF/s tf32 MMA) | fp64 DMMA {t64 * 1e6:8.1f} us "
          f"({K * n * n / t64 / 1e12:5.1f} TF/s) | speedup {t64 / t32:5.1f}x | max rel err {err:.2e}", flush=True)
