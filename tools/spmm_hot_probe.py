# Hot-row staged SpMM (lr_spmm_hot_f64) against the plain group kernel on the cfg4 rating shape:
# time (median of 8) and bit-identity of the results, per width and side.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device, sparse
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev, spmm_t_dev
o = workloads.cfg4()
A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix()
dp = A.pattern(); A.device_values()
for name, side in (("csr (columns)", dp.csr), ("csc (rows)", dp.csc)):
    h = side.hot()
    print(name, "hot encoding:", None if h is None else
          {hh: round(float(h[3][hh - 1]), 3) for hh in (64, 128, 256, 512, 1024, 1280, 2048, 4096) if hh <= h[2]}, flush=True)
rng = np.random.default_rng(0)
def med(fn):
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:])) * 1e3, out
for w in tuple(int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4,11,16,22,33,45,66,89,110,132,220".split(","))):
    X = device.to_device(rng.standard_normal((A.cols, w)))
    H = device.to_device(rng.standard_normal((A.rows, w)))
    line = []
    for name, fn in (("csr", lambda: spmm_dev(A, X)), ("csc", lambda: spmm_t_dev(A, H))):
        sparse.HOT_ROWS = True; sparse.HOT_MIN_SHARE = 0.0
        t_hot, y_hot = med(fn)
        for s in (dp.csr, dp.csc):
            keep = s._hot
        saved = (dp.csr._hot, dp.csc._hot)
        dp.csr._hot = dp.csc._hot = None
        t_plain, y_plain = med(fn)
        dp.csr._hot, dp.csc._hot = saved
        same = bool(torch.equal(y_hot, y_plain))
        line.append(f"{name} plain {t_plain:6.0f} hot {t_hot:6.0f} us ({t_plain / t_hot:4.2f}x) identical={same}")
    print(f"w={w:3d}: " + " | ".join(line), flush=True)
