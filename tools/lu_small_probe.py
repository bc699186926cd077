# one-CTA GEPP (the SVT loop's small Krylov blocks) vs CTA size (LR_LU_SMALL_THREADS)
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
out = []
for m, n in ((1000, 16), (1000, 21), (2048, 26), (1000, 64)):
    X = device.to_device(np.random.default_rng(m + n).standard_normal((m, n)))
    Y = device.empty(m, n)
    ts = []
    for it in range(12):
        Y.copy_(X); torch.cuda.synchronize(); t = time.perf_counter()
        linalg.lu_pl_dev(Y); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    out.append(f"{m}x{n} {np.median(ts[2:])*1e6:.1f} us")
print(" | ".join(out))
