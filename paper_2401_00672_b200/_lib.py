"""Thin ctypes binding of libpobk.so (include/pobk.h).  Argument marshalling only: every step of
the POBK path (preprocessing included) runs in the native library.  PyTorch is used for device
memory and streams; the library itself never sees a torch type.

There is no fallback: if libpobk.so is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpobk.so")

OK, ERR_ARG, ERR_BAD_CSR, ERR_ZERO_ROW, ERR_UNSTABLE_THR, ERR_CUDA, ERR_OOM, ERR_NO_DEVICE = range(8)
TERM_CONVERGED, TERM_MAX_SWEEPS, TERM_NONFINITE = 0, 1, 2
STOP = {"rse": 0, "relres": 1, "none": 2}
ORDER = {"schedule": 0, "residual": 1}
KERNEL = {"auto": 0, "launch": 1, "wavefront": 2, "smem": 3, "cluster": 4, "blocks": 5}
KERNEL_NAME = {v: k for k, v in KERNEL.items()}
TERM_NAME = {TERM_CONVERGED: "converged", TERM_MAX_SWEEPS: "max_sweeps", TERM_NONFINITE: "nonfinite"}


class PreprocessOpts(ctypes.Structure):
    _fields_ = [("thr", ctypes.c_double), ("reorder", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("tile_rows", ctypes.c_int32), ("guard", ctypes.c_int32)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_sweeps", ctypes.c_int64), ("stop", ctypes.c_int32),
                ("check_every", ctypes.c_int32), ("sweep_offset", ctypes.c_int64), ("order", ctypes.c_int32)]


class BlocksOpts(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("thr", ctypes.c_double), ("reorder", ctypes.c_int32)]


class LayoutStats(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("ntiles", ctypes.c_int32), ("nchunks", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("private_nnz_frac", ctypes.c_double),
                ("interior_row_frac", ctypes.c_double), ("stream_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["kernel"] = KERNEL_NAME.get(self.kernel, self.kernel)
        return d


class Report(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("termination", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("final_value", ctypes.c_double), ("solve_seconds", ctypes.c_double),
                ("sweep_seconds", ctypes.c_double), ("launches", ctypes.c_int64), ("sweeps_total", ctypes.c_int64),
                ("final_rse", ctypes.c_double), ("final_relres", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {"sweeps": int(self.sweeps), "termination": TERM_NAME.get(self.termination, self.termination),
                "kernel": KERNEL_NAME.get(self.kernel, self.kernel), "final_value": float(self.final_value),
                "solve_seconds": float(self.solve_seconds), "sweep_seconds": float(self.sweep_seconds),
                "launches": int(self.launches), "sweeps_total": int(self.sweeps_total),
                "final_rse": float(self.final_rse), "final_relres": float(self.final_relres)}


class PobkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pobk error {code}: {msg}")
        self.code = code


# symbol -> (restype, argtypes); the ABI declared in include/pobk.h
P = ctypes.c_void_p
I32, I64, F64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
SIGNATURES = {
    "pobk_preprocess_opts_default": (None, [ctypes.POINTER(PreprocessOpts)]),
    "pobk_solve_opts_default": (None, [ctypes.POINTER(SolveOpts)]),
    "pobk_preprocess": (I32, [I64, P, P, P, ctypes.POINTER(PreprocessOpts), ctypes.c_int, ctypes.POINTER(P)]),
    "pobk_plan_info": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32),
                             ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(F64)]),
    "pobk_plan_get_perm": (I32, [P, P]),
    "pobk_plan_get_partition": (I32, [P, P, P, P]),
    "pobk_plan_get_tiles": (I32, [P, ctypes.POINTER(I32), P]),
    "pobk_plan_get_layout_stats": (I32, [P, ctypes.POINTER(LayoutStats)]),
    "pobk_solve": (I32, [P, P, P, P, ctypes.POINTER(SolveOpts), P, ctypes.POINTER(Report)]),
    "pobk_solve_host": (I32, [P, P, P, P, ctypes.POINTER(SolveOpts), P, ctypes.POINTER(Report)]),
    "pobk_solve_batch": (I32, [ctypes.POINTER(P), I32, P, P, P, ctypes.POINTER(SolveOpts), P, P]),
    "pobk_solve_batch_host": (I32, [ctypes.POINTER(P), I32, P, P, P, ctypes.POINTER(SolveOpts), P, P]),
    "pobk_solve_multi": (I32, [P, I32, P, P, P, ctypes.POINTER(SolveOpts), P, P]),
    "pobk_residual_norm": (I32, [P, P, P, P, ctypes.POINTER(F64)]),
    "pobk_residual_sumsq_rows": (I32, [P, I64, I64, P, P, P, ctypes.POINTER(F64)]),
    "pobk_blocks_preprocess": (I32, [I64, P, P, P, ctypes.POINTER(BlocksOpts), ctypes.c_int, ctypes.POINTER(P)]),
    "pobk_blocks_info": (I32, [P, ctypes.POINTER(I32), P, P, P, ctypes.POINTER(I32), P, ctypes.POINTER(I32),
                               ctypes.POINTER(F64), ctypes.POINTER(F64)]),
    "pobk_plan_destroy": (None, [P]),
    "pobk_last_error": (ctypes.c_char_p, []),
    "pobk_abi_version": (I32, []),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2401_00672_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int):
    if status != OK:
        raise PobkError(status, lib.pobk_last_error().decode(errors="replace"))


def as_host(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(P)
