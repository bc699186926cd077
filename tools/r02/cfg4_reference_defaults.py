"""The REAL reference (/root/reference/pkg/src, build container only) on the
cfg4 rating shape at its own defaults: tau = 5n, delta = 1.2mn/nnz
(completion.py:328-335), eps = 0.17, reuse-q, i_reuse = 50 (cli.py:277-282),
split by its own split_observations(obs, 0.9, RngState(0)).  i_max = 1: the
first iteration already shows the blow-up (relative residual ~72: the top
singular direction of P(M) lives on rows/columns observed at densities up to
0.79, where a step of delta = 1.2/p ~ 247 overshoots by two orders of
magnitude); iteration 2's rank escalation then runs k past 2000 (the dense
cap) -- see profiles/r02_cfg4_defaults.txt for the GPU trace of that step.
Writes the trace to stdout."""
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
from lowrank.completion import SvtParams, svt_fast  # noqa: E402
from lowrank.ingest import split_observations  # noqa: E402
from lowrank.rng import RngState  # noqa: E402
from lowrank.sparse import ObservationSet  # noqa: E402

from paper_1810_06860_b200 import workloads  # noqa: E402

o = workloads.cfg4()
full = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
tagged, cold = split_observations(full, 0.9, RngState(0))
assert np.array_equal(tagged.split, o.split), "workloads.cfg4 split differs from the reference's split_observations"
print("split identical to the reference's split_observations; cold-start ids", cold, flush=True)
t = time.time()
res = svt_fast(tagged, SvtParams(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0,
                                 i_max=int(os.environ.get("IMAX", "1"))))
for tr in res.trace:
    print(f"reference i={tr.iteration} k={tr.k} r={tr.r} p={tr.p} q={tr.q} resid={tr.residual!r} {tr.svd_source} "
          f"{tr.wall_time:.1f}s", flush=True)
print(f"S = {res.S!r}  ({time.time() - t:.0f}s)")
