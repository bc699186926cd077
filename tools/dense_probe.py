import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
for m, n in ((100000, 110), (138493, 65), (1000, 16), (1000000, 305)):
    X = device.to_device(np.random.default_rng(m).standard_normal((m, n)))
    print(f"lu {m}x{n}: {timeit(lambda: linalg.lu_pl_dev(X, inplace=False)):.3f} ms", flush=True)
for n in (84, 260, 660, 1220):
    Xg = np.random.default_rng(n).standard_normal((3 * n, n)); G = Xg.T @ Xg
    def f():
        Gd = device.to_device(G); linalg.potrf_inv_dev(Gd)
    print(f"potrf_inv {n}: {timeit(f):.3f} ms", flush=True)
