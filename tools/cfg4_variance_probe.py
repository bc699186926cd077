# cfg4 SVT loop (bench settings) repeated in one process: per-run it/s and per-iteration wall times
import gc, os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o4 = workloads.cfg4()
obs4 = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
prm = completion.SvtParams(epsilon=0.17, i_reuse=5, q_reuse=10, strategy="reuse-q", seed=0, i_max=20,
                           delta=1.0, tau=5.0 * o4.n / 40)
NOGC = bool(os.environ.get("NOGC"))  # collect before each run and pause the collector inside it
for rep in range(5):
    if NOGC:
        gc.collect(); gc.disable()
    torch.cuda.synchronize()
    res = completion.svt_fast(obs4, prm)
    torch.cuda.synchronize()
    if NOGC:
        gc.enable()
    walls = [t.wall_time * 1e3 for t in res.trace]
    print(f"run {rep}: {res.iterations / (sum(walls) / 1e3):.1f} it/s; iteration ms: {[round(w, 1) for w in walls]}", flush=True)
