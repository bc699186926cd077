# Time lr_potrf_inv_f64 (with and without the inverse) at the orth widths.
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, device

lib = _native.load()
for n in tuple(int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["110", "330", "660", "1220", "2048"])):
    X = np.random.default_rng(n).standard_normal((4 * n, n))
    G0 = device.to_device(X.T @ X)
    G = device.empty(n, n)
    Rinv = device.empty(n, n)
    work = device.arena().get("pw", int(lib.lr_potrf_workspace_doubles(n)))
    info = ctypes.c_int(0)
    res = {}
    for label, rp in (("chol+inv", Rinv), ("chol", None)):
        ts = []
        for it in range(12):
            G.copy_(G0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.call("lr_potrf_inv_f64", n, device.ptr(G), device.ld(G), 0.0, device.ptr(rp), device.ld(Rinv),
                         device.ptr(work), None, device.stream())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[label] = np.median(ts[2:])
    R = device.to_host(G)
    err = np.linalg.norm(R.T @ R - X.T @ X) / np.linalg.norm(X.T @ X)
    print(f"n={n:5d} chol+inv {res['chol+inv']*1e3:8.1f} us  chol {res['chol']*1e3:8.1f} us  relerr {err:.1e}", flush=True)
