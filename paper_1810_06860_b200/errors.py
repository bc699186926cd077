"""Error taxonomy of the drop-in.

The class names and the inheritance tree are the reference's public contract
(/root/reference/pkg/src/lowrank/errors.py:7-28): callers catch them by name
and its CLI maps them to exit codes.  The native layer reports status codes
(include/lowrank_b200.h) that _native.check() turns into these types.
"""

__all__ = ["LowRankError", "RankDeficiencyError", "NumericalError", "SizeCapError", "DataError",
           "ConfigError"]


class LowRankError(Exception):
    """Root of every error raised by this package."""


class RankDeficiencyError(LowRankError):
    """A factorization needed full column rank and the device found it lost
    (LR_ERR_RANK, or a host-side check of a device-computed pivot/eigenvalue)."""


class NumericalError(LowRankError):
    """An iterative device solver (Jacobi sweeps) ran out of iterations
    (LR_ERR_NOCONV)."""


class SizeCapError(LowRankError):
    """The dense-SVD route was asked for min(m, n) above its cap."""


class DataError(LowRankError):
    """Input patterns, triples or observation sets are malformed."""


class ConfigError(LowRankError):
    """Run parameters are inconsistent."""
