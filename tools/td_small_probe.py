# syevd time at small n: single-warp tridiagonalization vs the CTA / cooperative kernels (LR_TD_WARP_MAX=0)
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
for n in ([int(a) for a in sys.argv[1:]] or (16, 32, 64, 84, 96, 110, 128)):
    X = np.random.default_rng(n).standard_normal((3 * n, n)); B = X.T @ X; G = device.to_device(B)
    for _ in range(2): linalg.sym_eig_dev(G)
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        t = time.perf_counter(); V, d = linalg.sym_eig_dev(G); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    dh = device.to_host(d); Vh = device.to_host(V); ref = np.linalg.eigvalsh(B)
    print(f"n={n}: {np.median(ts)*1e3:.3f} ms  eig err {np.max(np.abs(dh-ref))/ref[-1]:.1e} "
          f"resid {np.linalg.norm(B @ Vh - Vh * dh) / np.linalg.norm(B):.1e}", flush=True)
