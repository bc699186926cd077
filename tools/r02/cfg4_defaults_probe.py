"""cfg4 rating shape at the reference's own settings: tau = 5n, delta =
1.2mn/nnz (completion.py:328-335), the CLI rating defaults eps = 0.17,
reuse-q, i_reuse = 50, q_reuse = 10 (cli.py:277-282), seed 0.  Prints the
trace as it runs (LR_SVT_VERBOSE) and the pattern's density extremes."""
import os, sys, time
os.environ["LR_SVT_VERBOSE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet

t = time.time()
o = workloads.cfg4(**({"row_cap": int(os.environ["ROW_CAP"])} if "ROW_CAP" in os.environ else {}))
print(f"cfg4 generated in {time.time()-t:.1f}s", flush=True)
tr = o.split == 0
rc = np.bincount(o.rows[tr], minlength=o.m); cc = np.bincount(o.cols[tr], minlength=o.n)
print("train nnz", int(tr.sum()), "row nnz min/med/max", rc.min(), np.median(rc), rc.max(),
      "col nnz min/med/max", cc.min(), np.median(cc), cc.max(), "max col density", cc.max() / o.m, flush=True)
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
imax = int(os.environ.get("IMAX", "500"))
p = completion.SvtParams(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax)
t = time.time()
try:
    res = completion.svt_fast(obs, p)
    rt, ct, vt = obs.subset(1)
    print(f"done {res.iterations} it conv={res.converged} resid={res.residual:.6e} rank={res.rank} "
          f"{time.time()-t:.1f}s MAE={completion.mae(res.predict(rt, ct), vt):.6f}", flush=True)
except Exception as e:
    print("FAILED", type(e).__name__, str(e)[:300], f"after {time.time()-t:.1f}s", flush=True)
