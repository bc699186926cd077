"""Round-2 probe: where do the long recycling traces leave the reference's?
Prints, per golden trace, the per-iteration relative residual difference and
the first iteration whose k/r/p/q/source differ."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet

g = dict(np.load("tests/golden/reference_golden.npz"))


def report(name, got, prefix):
    rr = g[prefix + "residual"]
    n = min(len(rr), got.iterations)
    res = np.array([t.residual for t in got.trace[:n]])
    d = np.abs(res - rr[:n]) / rr[:n]
    fd = [int(np.argmax(d > t)) if (d > t).any() else n for t in (1e-13, 1e-10, 1e-8, 1e-6)]
    disc = next((i for i, t in enumerate(got.trace[:n]) if (t.k, t.r, t.p, t.q, t.svd_source) !=
                 (g[prefix + "k"][i], g[prefix + "r"][i], g[prefix + "p"][i], g[prefix + "q"][i], g[prefix + "source"][i])), n)
    print(f"{name}: ours {got.iterations} it conv={got.converged} resid={got.residual:.6e} | ref {len(rr)} it "
          f"conv={bool(g[prefix+'converged'])} resid={rr[-1]:.6e} | first rel diff >1e-13,1e-10,1e-8,1e-6 at {fd}; "
          f"first discrete diff at {disc}", flush=True)
    for i in list(range(0, min(n, 200), 10)):
        print(f"   i={i+1} d={d[i]:.2e} ours(k,r,p,q)={got.trace[i].k, got.trace[i].r, got.trace[i].p, got.trace[i].q} "
              f"ref={g[prefix+'k'][i], g[prefix+'r'][i], g[prefix+'p'][i], g[prefix+'q'][i]}")
    if disc < n:
        i = disc
        print(f"   discrete diff at i={i+1}: ours {got.trace[i]} ref k={g[prefix+'k'][i]} r={g[prefix+'r'][i]} "
              f"p={g[prefix+'p'][i]} q={g[prefix+'q'][i]} src={g[prefix+'source'][i]} resid={rr[i]:.16e}")
        if i > 0:
            print(f"   previous residuals ours {got.trace[i-1].residual:.16e} ref {rr[i-1]:.16e}")


ob2 = ObservationSet(100, 100, g["tc_rows"], g["tc_cols"], g["tc_vals"])
report("tc_rq", completion.svt_fast(ob2, completion.SvtParams(epsilon=1e-2, seed=7, strategy="reuse-q", i_reuse=25)), "tc_rq_")
o, _ = workloads.cfg1_small()
ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
report("small_rq", completion.svt_fast(ob, completion.SvtParams(epsilon=1e-3, seed=4, strategy="reuse-q", i_reuse=20)), "svt_small_rq_")
report("small_ru", completion.svt_fast(ob, completion.SvtParams(epsilon=1e-3, seed=4, strategy="reuse-u", i_reuse=20)), "svt_small_ru_")
