# Time the device eigensolvers and dense pieces at BKI-relevant sizes.
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
for method in ("syevd", "syevj"):
    linalg.EIG_METHOD = method
    for n in (2, 3, 11, 84, 96, 130, 260, 660, 1300):
        if method == "syevj" and n > 700: continue
        X = np.random.default_rng(n).standard_normal((3 * n, n))
        B = X.T @ X
        G = device.to_device(B)
        linalg.sym_eig_dev(G); torch.cuda.synchronize()
        t = time.perf_counter(); V, d = linalg.sym_eig_dev(G); torch.cuda.synchronize(); dt = time.perf_counter() - t
        ref = np.linalg.eigvalsh(B)
        dh = device.to_host(d); Vh = device.to_host(V)
        orth = np.linalg.norm(Vh.T @ Vh - np.eye(n)); resid = np.linalg.norm(B @ Vh - Vh * dh) / np.linalg.norm(B)
        print(f"{method} n={n}: {dt*1e3:.2f} ms, eig err {np.max(np.abs(dh-ref))/ref[-1]:.2e} orth {orth:.1e} resid {resid:.1e}", flush=True)
# degenerate spectrum (clusters)
linalg.EIG_METHOD = "syevd"
Q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((300, 300)))
ev = np.concatenate([np.full(100, 1.0), np.linspace(2, 3, 150), np.full(50, 5.0)])
B = (Q * ev) @ Q.T; B = 0.5 * (B + B.T)
V, d = linalg.sym_eig_dev(device.to_device(B)); Vh = device.to_host(V); dh = device.to_host(d)
print("clustered 300:", np.max(np.abs(dh - np.sort(ev))), np.linalg.norm(Vh.T @ Vh - np.eye(300)), np.linalg.norm(B @ Vh - Vh * dh))
for n in (84, 660):
    X = np.random.default_rng(n).standard_normal((3 * n, n))
    Gd = device.to_device(X.T @ X)
    torch.cuda.synchronize(); t = time.perf_counter(); info, Ri = linalg.potrf_inv_dev(Gd); torch.cuda.synchronize(); print(f"potrf_inv n={n}: {(time.perf_counter()-t)*1e3:.2f} ms")
