"""ctypes loader for libganq.so (the C ABI of include/ganq.h).

Argument marshalling only: every step of the solver runs in the CUDA kernels of
libganq.so.  There is no CPU or PyTorch fallback -- if the library is missing or
fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libganq.so")

_lock = threading.Lock()
_lib = None

OK, ERR_INVALID_ARG, ERR_NOT_PD, ERR_CUDA, ERR_WORKSPACE, ERR_UNSUPPORTED = range(6)
PRECOND = {"adaptive": 0, "fixed_lambda": 1, "none": 2}

# symbol -> (restype, argtypes); must match include/ganq.h
P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
SIG = {
    "ganq_default_opts": (None, [P]),
    "ganq_hessian": (I32, [P, I64, I64, P, I32, P]),
    "ganq_hessian_workspace_size": (ctypes.c_size_t, [I64, I64]),
    "ganq_hessian_ws": (I32, [P, I64, I64, P, I32, P, ctypes.c_size_t, P]),
    "ganq_hessian_fixed_size": (ctypes.c_size_t, [I64]),
    "ganq_hessian_partials_size": (ctypes.c_size_t, [I64, I64]),
    "ganq_hessian_partials": (I32, [P, I64, I64, P, P, P]),
    "ganq_hessian_fixed": (I32, [P, I64, I64, P, P, I32, P]),
    "ganq_hessian_finalize": (I32, [P, P, I64, P, I32, P]),
    "ganq_workspace_size": (ctypes.c_size_t, [I64, I64, I32]),
    "ganq_quantize_layer": (I32, [P, I64, I64, P, I32, I32, P, P, P, P, ctypes.c_size_t, P]),
    "ganq_objective_workspace_size": (ctypes.c_size_t, [I64, I64]),
    "ganq_objective": (I32, [P, P, P, P, I64, I64, I32, P, P, P, ctypes.c_size_t, P]),
    "ganq_tstep": (I32, [P, P, P, I64, I64, I32, I32, P, P, P, ctypes.c_size_t, P]),
    "ganq_factor": (I32, [P, I64, P, P, P, P, ctypes.c_size_t, P]),
    "ganq_profile_enable": (I32, [I32]),
    "ganq_profile_read": (I32, [P, P, I32]),
    "ganq_profile_stage_name": (ctypes.c_char_p, [I32]),
    "ganq_launch_count": (I64, []),
    "ganq_last_error": (ctypes.c_char_p, []),
    "ganq_last_error_index": (I64, []),
    "ganq_version": (ctypes.c_char_p, []),
    "ganq_packed_row_bytes": (I64, [I64, I32]),
    "ganq_pack_codes": (I32, [P, I64, I64, I32, P, P]),
    "ganq_codebook_f16": (I32, [P, I64, I32, P, P]),
    "ganq_lut_gemm": (I32, [P, P, P, I64, I64, I64, I32, P, P]),
    "ganq_outlier_split": (I32, [P, I64, I64, ctypes.c_double, P, P, P, P, P, P]),
    "ganq_outlier_csr": (I32, [P, I64, I64, P, P, P, P, P, P]),
    "ganq_sparse_gemm_add": (I32, [P, P, P, I64, I64, P, I64, P, P]),
    "ganq_kmeans_codebook": (I32, [P, I64, I64, I32, I32, P, P]),
}


class Opts(ctypes.Structure):
    """ganq_opts_t (include/ganq.h)."""
    _fields_ = [
        ("precond", ctypes.c_int32),
        ("empty_level_rule", ctypes.c_int32),
        ("lam", ctypes.c_double),
        ("tau", ctypes.c_double),
        ("T0", ctypes.c_void_p),
        ("obj_trace", ctypes.POINTER(ctypes.c_double)),
    ]


class GanqError(RuntimeError):
    def __init__(self, status: int, msg: str, index: int = -1):
        super().__init__(f"ganq status {status}: {msg}")
        self.status = status
        self.index = index


class NotPositiveDefinite(GanqError):
    pass


def load(path: str = LIB_PATH):
    """Load libganq.so (building it first if the sources are newer); raise if impossible."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            try:
                from . import build as _build
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise RuntimeError(f"libganq.so missing at {path} and could not be built: {e}") from e
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIG.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == OK:
        return
    lib = load()
    msg = lib.ganq_last_error().decode(errors="replace")
    idx = int(lib.ganq_last_error_index())
    if status == ERR_NOT_PD:
        raise NotPositiveDefinite(status, msg, idx)
    raise GanqError(status, msg, idx)
