"""Per-call CUDA-event timing of the native kernels and their roofline
models.

Algorithmic bytes / flops per launch (fp64 = 8 B, int32 = 4 B):
  spmm   (rows r, cols c, width w, nnz):  B = 12 nnz + 4 (r+1) + 8 c w + 8 r w,
                                          F = 2 nnz w
  svt step (m, n, rank r, nnz):           B = 4 (m+1) + 28 nnz + 8 (m+n) r + 8 r,
                                          F = 2 r nnz + 4 nnz
        per entry: column index 4, M 8, Y (CSR) read + write 16; with the
        in-step CSC scatter (completion.CSC_SCATTER) + 12 (inverse perm 4,
        CSC store 8) = SURVEY 8(d)'s 40 B/nnz
  csc refresh (lr_gather_f64, nnz):       B = 20 nnz (perm 4, CSR value 8, CSC store 8)
  gemm   (M, N, K):                       F = 2 M N K  (SYRK: M (M+1) K, one triangle),
                                          B = 8 (M K + K N + M N)
The dense kernels are bound by the fp64 tensor peak, the sparse ones by HBM
on compulsory bytes; GEPP / Jacobi / Cholesky are latency-bound and reported
as time and share only.
"""

from __future__ import annotations

from collections import defaultdict

import torch


def spmm_model(meta):
    """fp64: value 8 B + index 4 B per entry; fp32 mode (bytes_per_value 4):
    value 4 B + index 4 B and 4 B per dense element."""
    nnz, r, c, w = meta["nnz"], meta["rows"], meta["cols"], meta["w"]
    b = meta.get("bytes_per_value", 8)
    return (b + 4) * nnz + 4 * (r + 1) + b * c * w + b * r * w, 2 * nnz * w


def svt_model(meta):
    nnz, m, n, r = meta["nnz"], meta["m"], meta["n"], meta["r"]
    per = 40 if meta.get("csc_scatter", True) else 28
    return 4 * (m + 1) + per * nnz + 8 * (m + n) * r + 8 * r, 2 * r * nnz + 4 * nnz


def gather_model(meta):
    nnz = meta["nnz"]
    return 20 * nnz, 0


def gemm_model(meta):
    M, N, K = meta["M"], meta["N"], meta["K"]
    syrk = bool(meta.get("flags", 0) & 2)
    bupper = bool(meta.get("flags", 0) & 1)
    flops = M * (M + 1) * K if syrk else (M * N * K if bupper else 2 * M * N * K)
    return 8 * (M * K + K * N + M * N), flops


MODELS = {"lr_spmm_f64": ("hbm", spmm_model), "lr_spmm_f32": ("hbm", spmm_model),
          "lr_spmm_hot_f64": ("hbm", spmm_model),
          "lr_svt_step_f64": ("hbm", svt_model), "lr_svt_step_flat_f64": ("hbm", svt_model), "lr_gather_f64": ("hbm", gather_model),
          "lr_gemm_f64": ("tensor", gemm_model)}


def gather_bytes(name, meta):
    """Diagnostic L2-gather bytes: one dense row of w (SpMM) or r
    (SVT step) values per stored entry."""
    if meta is None:
        return 0
    if name in ("lr_spmm_f64", "lr_spmm_f32", "lr_spmm_hot_f64"):
        return meta.get("bytes_per_value", 8) * meta["nnz"] * meta["w"]
    if name in ("lr_svt_step_f64", "lr_svt_step_flat_f64"):
        return 8 * meta["nnz"] * meta["r"]
    return 0


class Profiler:
    """Records a (start, end) CUDA event pair around every native call."""

    def __init__(self):
        self.records = []

    def run(self, name, meta, fn, args):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = fn(*args)
        e1.record()
        self.records.append((name, meta, e0, e1))
        return st

    def summary(self):
        torch.cuda.synchronize()
        out = defaultdict(lambda: {"calls": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0, "modeled_ms": 0.0,
                                   "gather": 0.0})
        for name, meta, e0, e1 in self.records:
            ms = e0.elapsed_time(e1)
            d = out[name]
            d["calls"] += 1
            d["ms"] += ms
            if name in MODELS and meta is not None:
                b, f = MODELS[name][1](meta)
                d["bytes"] += b
                d["flops"] += f
                d["gather"] += gather_bytes(name, meta)
                d["modeled_ms"] += ms
        return dict(out)
