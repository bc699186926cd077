# Per-iteration wall time of the cfg4 job (third run), with k, r, p, source: where the job's time goes by phase.
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o4 = workloads.cfg4()
obs = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
params = bench.cfg4_params()
eng = completion.DeviceEngine(obs)
for _ in range(3):
    res = completion._svt_loop(obs, params, "rsvd-bki", params.strategy, engine=eng)
torch.cuda.synchronize()
tot = 0.0
for t in res.trace:
    tot += t.wall_time
    print(f"i={t.iteration:3d} k={t.k:3d} r={t.r:3d} p={t.p} q={t.q:2d} {t.svd_source:10s} {1e3 * t.wall_time:7.2f} ms  cum {1e3 * tot:7.1f}")
