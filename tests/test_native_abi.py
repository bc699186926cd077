"""CPU-side checks of the drop-in boundary: the C-ABI library loads (no GPU
needed to dlopen it) and exports every symbol include/lowrank_b200.h
declares, with a ctypes signature for each."""

import os
import re

import pytest

from paper_1810_06860_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lowrank_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared_symbols()
    for must in ("lr_spmm_f64", "lr_svt_step_f64", "lr_gemm_f64", "lr_lu_pl_f64", "lr_syevj_f64",
                 "lr_potrf_inv_f64", "lr_gaussian_f64"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.fail(f"native library not built: {_native.LIB_PATH} (run make)")
    lib = _native.load()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.lr_version() >= 1


def test_ctypes_table_matches_header():
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_status_mapping():
    from paper_1810_06860_b200.errors import NumericalError, RankDeficiencyError

    _native.check(_native.LR_OK)
    with pytest.raises(ValueError):
        _native.check(_native.LR_ERR_ARG)
    with pytest.raises(RankDeficiencyError):
        _native.check(_native.LR_ERR_RANK)
    with pytest.raises(NumericalError):
        _native.check(_native.LR_ERR_NOCONV)
    with pytest.raises(RuntimeError):
        _native.check(_native.LR_ERR_CUDA)


def test_argument_errors_without_gpu():
    # shape validation happens before any device work
    lib = _native.load()
    assert lib.lr_gemm_f64(0, 4, 4, 4, 1.0, None, 1, None, 4, 0.0, None, 4, 0, None, 0, None) == _native.LR_ERR_ARG
    assert "leading" in _native.last_error()
    assert lib.lr_lu_pl_f64(3, 5, None, 5, None, None, None) == _native.LR_ERR_ARG
    assert "m >= n" in _native.last_error()
