import sys, numpy as np
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
rng = np.random.default_rng(0)
for rep in range(3):
    for (M, N, K) in ((120, 5, 8), (120, 8, 8), (64, 5, 8), (200, 5, 8), (120, 5, 16)):
        A = rng.standard_normal((M, K)); B = rng.standard_normal((K, N))
        C = device.to_host(linalg.matmul_dev(device.to_device(A), device.to_device(B)))
        err = np.abs(C - A @ B).max()
        zr = np.flatnonzero(np.all(C == 0, axis=1))
        print(rep, (M, N, K), "err", err, "zero rows", zr.size, zr[:4], flush=True)
