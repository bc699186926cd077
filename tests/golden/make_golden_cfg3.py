"""Golden SVT trace of the REAL reference on cfg3 (the image-inpainting shape,
SURVEY.md 8(d) recorded variant), written to tests/golden/reference_golden_cfg3.npz.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_cfg3.py

Stored: the trace (k, r, p, q, residual, source), S, and U/V rounded to the
top few singular vectors' sign-fixed projections are NOT stored (the factors
are 2048 x r; the test compares S, the trace and predictions at a fixed
sample of cells instead).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from lowrank.completion import SvtParams, svt_fast  # noqa: E402
from lowrank.sparse import ObservationSet  # noqa: E402

from paper_1810_06860_b200 import workloads  # noqa: E402


def main():
    o, _ = workloads.cfg3()
    ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
    res = svt_fast(ob, SvtParams(strategy="reuse-u", i_reuse=100, q_reuse=10, seed=0, epsilon=0.05))
    t = res.trace
    rng = np.random.default_rng(123)
    pr, pc = rng.integers(0, o.m, 5000), rng.integers(0, o.n, 5000)
    g = {"k": np.array([x.k for x in t]), "r": np.array([x.r for x in t]), "p": np.array([x.p for x in t]),
         "q": np.array([x.q for x in t]), "residual": np.array([x.residual for x in t]),
         "source": np.array([x.svd_source for x in t]), "S": res.S, "converged": np.array(res.converged),
         "pred_rows": pr, "pred_cols": pc, "pred": res.predict(pr, pc)}
    np.savez_compressed(os.path.join(HERE, "reference_golden_cfg3.npz"), **g)
    print({k: (v if v.size < 8 else v.shape) for k, v in g.items()})


if __name__ == "__main__":
    main()
