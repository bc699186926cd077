import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
for n in (260, 660, 1300):
    X = np.random.default_rng(n).standard_normal((3 * n, n))
    G = device.to_device(X.T @ X)
    linalg.sym_eig_dev(G); torch.cuda.synchronize()
    t = time.perf_counter(); V, d = linalg.sym_eig_dev(G); torch.cuda.synchronize()
    print(sys.argv[1], n, f"{(time.perf_counter()-t)*1e3:.2f} ms", flush=True)
