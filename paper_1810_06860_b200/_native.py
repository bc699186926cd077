"""ctypes binding of the C ABI in include/lowrank_b200.h.

The library is built in-tree (`make`, or `__graft_entry__.build()`) into
paper_1810_06860_b200/_native/liblowrank_b200.so.  There is no CPU fallback:
if the library or a CUDA device is missing, every numerical entry point
raises instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NumericalError, RankDeficiencyError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LR_NATIVE_LIB") or os.path.join(_HERE, "_native", "liblowrank_b200.so")  # override: experiments only

LR_OK, LR_ERR_ARG, LR_ERR_RANK, LR_ERR_NOCONV, LR_ERR_CUDA = 0, 1, 2, 3, 4
LR_GEMM_B_UPPER, LR_GEMM_SYRK_UPPER = 1, 2

_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong
_D = ctypes.c_double
_ULL = ctypes.c_ulonglong

# name -> (restype, argtypes); mirrors include/lowrank_b200.h
SIGNATURES = {
    "lr_version": (_I, []),
    "lr_last_error": (ctypes.c_char_p, []),
    "lr_sm_count": (_I, []),
    "lr_launch_count": (_LL, []),
    "lr_spmm_f64": (_I, [_P, _P, _P, _I, _P, _I, _P, _I, _P, _LL, _I, _P, _LL, _P, _P]),
    "lr_spmm_hot_rows_max": (_I, []),
    "lr_spmm_hot_buf_doubles": (_LL, []),
    "lr_spmm_hot_f64": (_I, [_P, _P, _P, _P, _I, _P, _LL, _P, _I, _P, _I, _P, _I, _P, _LL, _I, _P, _LL, _P, _P]),
    "lr_spmm_f32": (_I, [_P, _P, _P, _I, _P, _I, _P, _I, _P, _LL, _I, _P, _LL, _P, _P]),
    "lr_csr_transpose_workspace_ints": (_LL, [_I, _I]),
    "lr_csr_transpose_i32": (_I, [_I, _I, _LL, _P, _P, _P, _P, _P, _P, _P, _LL, _P]),
    "lr_sddmm_f64": (_I, [_P, _P, _I, _P, _I, _P, _LL, _P, _P, _LL, _I, _P, _P]),
    "lr_svt_step_f64": (_I, [_P, _P, _I, _P, _I, _P, _LL, _P, _P, _LL, _I, _P, _P, _P, _P, _D, _I,
                             _P, _I, _P, _P]),
    "lr_svt_step_partials": (_I, []),
    "lr_svt_tile_entries": (_I, []),
    "lr_svt_tile_count": (_LL, [_LL]),
    "lr_svt_tile_rows_i32": (_I, [_P, _I, _LL, _P, _P]),
    "lr_svt_flat_partials": (_I, []),
    "lr_svt_step_flat_f64": (_I, [_P, _P, _I, _LL, _P, _P, _LL, _P, _P, _LL, _I, _P, _P, _P, _P, _D, _I, _P, _I,
                                  _P, _P]),
    "lr_sddmm_flat_f64": (_I, [_P, _P, _I, _LL, _P, _P, _LL, _P, _P, _LL, _I, _P, _P]),
    "lr_pattern_axpy_f64": (_I, [_P, _P, _P, _P, _D, _LL, _P]),
    "lr_gather_f64": (_I, [_P, _P, _P, _LL, _P]),
    "lr_block_stats_f64": (_I, [_P, _LL, _LL, _LL, _P, _P, _P]),
    "lr_stats_partials": (_I, []),
    "lr_dot_f64": (_I, [_P, _P, _LL, _P, _P, _P]),
    "lr_power_update_f64": (_I, [_P, _P, _LL, _D, _P, _P, _P]),
    "lr_gemm_workspace_doubles": (_LL, [_I, _I, _I, _I, _I]),
    "lr_gemm_f64": (_I, [_I, _I, _I, _I, _D, _P, _LL, _P, _LL, _D, _P, _LL, _I, _P, _LL, _P]),
    "lr_potrf_workspace_doubles": (_LL, [_I]),
    "lr_potrf_inv_f64": (_I, [_I, _P, _LL, _D, _P, _LL, _P, _P, _P]),
    "lr_potrf_inv_async_f64": (_I, [_I, _P, _LL, _D, _P, _LL, _P, _P, _P]),
    "lr_lu_workspace_doubles": (_LL, [_I, _I]),
    "lr_lu_pl_f64": (_I, [_I, _I, _P, _LL, _P, _P, _P]),
    "lr_lu_pl_async_f64": (_I, [_I, _I, _P, _LL, _P, _P, _P]),
    "lr_syevj_workspace_doubles": (_LL, [_I]),
    "lr_syevj_f64": (_I, [_I, _P, _LL, _P, _P, _LL, _I, _P, _P, _P]),
    "lr_syevd_workspace_doubles": (_LL, [_I]),
    "lr_syevd_f64": (_I, [_I, _P, _LL, _P, _P, _LL, _P, _P, _P]),
    "lr_fix_signs_f64": (_I, [_P, _LL, _I, _I, _P, _LL, _I, _P]),
    "lr_scale_columns_f64": (_I, [_P, _LL, _I, _P, _I, _P, _I, _P, _LL, _P]),
    "lr_gram_spectrum_f64": (_I, [_P, _I, _P, _P]),
    "lr_gram_tf32x3_workspace_floats": (_LL, [_I, _I]),
    "lr_gram_tf32x3": (_I, [_P, _LL, _I, _I, _P, _LL, _P, _LL, _P]),
    "lr_coo_to_csr_workspace_ints": (_LL, [_I, _LL]),
    "lr_coo_to_csr_i32": (_I, [_I, _I, _LL, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _LL, _P, _P]),
    "lr_jacobi_sweep_f64": (_I, [_I, _I, _P, _LL, _P, _LL, _D, _D, _P, _P]),
    "lr_row_norms_f64": (_I, [_P, _LL, _I, _I, _P, _P]),
    "lr_gaussian_f64": (_I, [_ULL, _I, _I, _P, _LL, _P]),
    "lr_omega_assemble_f64": (_I, [_P, _P, _LL, _I, _I, _P, _LL, _P]),
    "lr_host_uniforms": (None, [_ULL, _LL, _LL, _P]),
    "lr_host_box_muller": (None, [_P, _P, _LL, _P]),
    "lr_host_cossin": (None, [_P, _LL, _P]),
    "lr_host_bm_assemble": (None, [_P, _P, _LL, _P]),
    "lr_convert_f64_to_f32": (_I, [_P, _LL, _P, _LL, _LL, _LL, _P]),
    "lr_convert_f32_to_f64": (_I, [_P, _LL, _P, _LL, _LL, _LL, _P]),
    "lr_copy2d_f64": (_I, [_P, _LL, _P, _LL, _LL, _LL, _I, _P]),
    "lr_fill_f64": (_I, [_P, _LL, _LL, _LL, _D, _P]),
    "lr_transpose_f64": (_I, [_P, _LL, _LL, _LL, _P, _LL, _P]),
    "lr_symmetrize_f64": (_I, [_P, _LL, _I, _P, _LL, _P]),
    "lr_diag_f64": (_I, [_P, _LL, _I, _P, _P]),
}

_lib = None


def load():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library missing: {LIB_PATH}. Build it with `make` (or "
                "__graft_entry__.build()); the B200 path has no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().lr_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == LR_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == LR_ERR_ARG:
        raise ValueError(msg)
    if status == LR_ERR_RANK:
        raise RankDeficiencyError(msg)
    if status == LR_ERR_NOCONV:
        raise NumericalError(msg)
    raise RuntimeError(msg)


PROFILER = None  # set to a profiling.Profiler to time every call with CUDA events


def call(name: str, *args, meta=None):
    """Invoke lr_<name> and map its status to the reference's exceptions.
    `meta` (shape facts) is only used by an active profiler."""
    fn = getattr(load(), name)
    if PROFILER is None:
        st = fn(*args)
    else:
        st = PROFILER.run(name, meta, fn, args)
    check(st, name)
    return st
