"""tc_rq (the reference's own reuse-q test case, chaotic after ~80
iterations; the reference takes dense fallbacks at i = 159 and 170): our
iteration count, events and discrete divergence from the golden trace under
the dense-SVD null floor given by LR_DENSE_NULL_FLOOR."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1810_06860_b200 import completion, linalg
from paper_1810_06860_b200.sparse import ObservationSet

g = dict(np.load("tests/golden/reference_golden.npz"))
ob = ObservationSet(100, 100, g["tc_rows"], g["tc_cols"], g["tc_vals"])
r = completion.svt_fast(ob, completion.SvtParams(epsilon=1e-2, seed=7, strategy="reuse-q", i_reuse=25))
p = "tc_rq_"
n = min(r.iterations, len(g[p + "k"]))
disc = next((i for i, t in enumerate(r.trace[:n]) if (t.k, t.r, t.p, t.q, t.svd_source) !=
             (g[p + "k"][i], g[p + "r"][i], g[p + "p"][i], g[p + "q"][i], g[p + "source"][i])), n)
print(f"floor={linalg.DENSE_NULL_FLOOR:g}: {r.iterations} iterations (ref 178), first discrete diff at "
      f"{disc + 1}, events {r.events}", flush=True)
