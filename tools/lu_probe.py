import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
X = device.to_device(np.random.default_rng(0).standard_normal((100000, 110)))
Y = device.empty(100000, 110)
def f():
    linalg._native.call("lr_copy2d_f64", device.ptr(X), device.ld(X), device.ptr(Y), device.ld(Y), 100000, 110, 0, device.stream())
    linalg.lu_pl_dev(Y)
f(); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): f()
torch.cuda.synchronize()
print(sys.argv[1] if len(sys.argv) > 1 else "", f"lu 100000x110: {(time.perf_counter()-t)/5*1e3:.3f} ms")
