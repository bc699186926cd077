# syevd time vs rows per CTA of the cooperative tridiagonalization (LR_TD_ROWS), at BKI-relevant n
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
out = []
for n in (130, 260, 660, 1300):
    X = np.random.default_rng(n).standard_normal((3 * n, n)); G = device.to_device(X.T @ X)
    for _ in range(2): linalg.sym_eig_dev(G)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        t = time.perf_counter(); linalg.sym_eig_dev(G); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    out.append(f"n={n} {np.median(ts)*1e3:.3f}")
print(" | ".join(out))
