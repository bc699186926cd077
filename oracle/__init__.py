"""CPU oracle for the SVT / rSVD-BKI / rSVD-PI hot path — TEST INFRASTRUCTURE ONLY.

This package is a from-scratch numpy/scipy restatement of the reference
package `lowrank` (arxiv 1810.06860, `/root/reference/pkg/src/lowrank`) for
exactly the functions on the north-star path.  It exists so that

* `tests/` can check the CUDA path against it on the same seeded inputs,
* `__graft_entry__.smoke()` can check one small GPU invocation, and
* `bench.py` can time the reference CPU algorithm on the GPU box host
  (`cpu_baseline`, kind "port", and the `--impl reference` arm).

Nothing in `paper_1810_06860_b200/` imports it: the product path has no CPU
fallback and fails loudly without its CUDA library.

Parity of this oracle is PINNED: `tests/test_oracle_golden.py` compares it
with `tests/golden/*.npz`, which `tests/golden/make_golden.py` produced by
importing the real reference package from `/root/reference/pkg/src` in the
build container (numpy 2.3.5 / scipy 1.18.1 / OpenBLAS 0.3.30).  The
arithmetic of the reference lives in third-party code that is not under
/root/reference (scipy sparsetools `csr_matvecs`, LAPACK dgeqrf/dorgqr,
dgetrf, dsyevd, dgesdd, numpy Philox); the oracle calls the same routines.
"""

from .philox_stream import Stream, gaussian_block
from .csr import (
    Pattern,
    csr_from_triples,
    csr_times_dense,
    csr_t_times_dense,
    sampled_product,
    scaled_norm,
    spectral_estimate,
)
from .dense import (
    RankDeficient,
    NoConvergence,
    SizeCap,
    Triplets,
    gram_svd,
    householder_basis,
    pivoted_lower,
    dense_svd,
)
from .sketch import SketchParams, Basis, sketch_pi, sketch_bki, sketch_basic, relative_fit_error
from .svt import SvtConfig, complete, run_power_rule

__all__ = [
    "Stream", "gaussian_block", "Pattern", "csr_from_triples", "csr_times_dense",
    "csr_t_times_dense", "sampled_product", "scaled_norm", "spectral_estimate",
    "RankDeficient", "NoConvergence", "SizeCap", "Triplets", "gram_svd",
    "householder_basis", "pivoted_lower", "dense_svd", "SketchParams", "Basis",
    "sketch_pi", "sketch_bki", "sketch_basic", "relative_fit_error", "SvtConfig",
    "complete", "run_power_rule",
]
