"""fp64 CPU oracle for GANQ (arxiv 2501.12956) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It shares no code with the
CUDA path (``paper_2501_12956_b200``); neither imports the other.  The only
module both sides use is ``synthetic`` (seeded input generators, no method
arithmetic).

The arithmetic lives in ``ganq_oracle.c`` (plain C, fp64, OpenMP over rows);
this file only marshals numpy arrays through ctypes.  Each wrapper names the
paper passage its C function follows (P:n = /root/reference/PAPER.md line n).

Parity status: every function is pinned by tests/test_oracle_pins.py
(see DESIGN.md "Oracle pins"); the per-iteration trajectory on realistic
data has no printed value in the paper and is "parity unpinned" beyond the
invariants (row "trajectory").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ganq_oracle.c")
_LIB = os.path.join(_HERE, "libganq_oracle.so")
_lock = threading.Lock()
_lib = None

PRECOND = {"adaptive": 0, "fixed_lambda": 1, "none": 2}
DEFAULT_TAU = 1e-7  # reading R-3: jitter tau * mean(diag H) on every delta_i


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc, -fopenmp, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.or_hessian_bf16.argtypes = [P, I64, I64, P]
        lib.or_hessian_bf16.restype = ctypes.c_int
        lib.or_precondition.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, ctypes.c_double, P, P]
        lib.or_precondition.restype = ctypes.c_int
        lib.or_cholesky.argtypes = [P, I64, P]
        lib.or_cholesky.restype = I64
        lib.or_pack.argtypes = [P, I64, I64, ctypes.c_int, P]
        lib.or_pack.restype = I64
        lib.or_unpack.argtypes = [P, I64, I64, ctypes.c_int, P]
        lib.or_unpack.restype = None
        lib.or_lut_gemm.argtypes = [P, P, P, I64, I64, I64, ctypes.c_int, P]
        lib.or_lut_gemm.restype = None
        lib.or_storage_bytes.argtypes = [I64, I64, ctypes.c_int, ctypes.c_int]
        lib.or_storage_bytes.restype = ctypes.c_double
        lib.or_outlier_indices.argtypes = [I64, ctypes.c_double, P, P]
        lib.or_outlier_indices.restype = None
        lib.or_outlier_split.argtypes = [P, I64, I64, ctypes.c_double, P, P, P, P]
        lib.or_outlier_split.restype = None
        lib.or_sparse_matmul.argtypes = [P, P, P, I64, I64, P, I64, P]
        lib.or_sparse_matmul.restype = None
        lib.or_kmeans_codebook.argtypes = [P, I64, I64, ctypes.c_int, ctypes.c_int, P]
        lib.or_kmeans_codebook.restype = None
        lib.or_init_codebook.argtypes = [P, I64, I64, ctypes.c_int, P]
        lib.or_init_codebook.restype = None
        lib.or_sstep.argtypes = [P, P, P, I64, I64, ctypes.c_int, P, P]
        lib.or_sstep.restype = None
        lib.or_sstep_audit.argtypes = [P, P, P, P, I64, I64, ctypes.c_int, P, P]
        lib.or_sstep_audit.restype = None
        lib.or_tstep.argtypes = [P, P, P, I64, I64, ctypes.c_int, ctypes.c_int, P, P, P, P]
        lib.or_tstep.restype = ctypes.c_int
        lib.or_objective.argtypes = [P, P, P, P, I64, I64, ctypes.c_int, P]
        lib.or_objective.restype = ctypes.c_double
        lib.or_quantize.argtypes = [P, I64, I64, P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double, P, ctypes.c_int, P, P, P]
        lib.or_quantize.restype = I64
        _lib = lib
        return lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class NotPositiveDefinite(RuntimeError):
    def __init__(self, index):
        super().__init__(f"cholesky: non-positive pivot at {index}")
        self.index = int(index)


def hessian_bf16(X_bits: np.ndarray) -> np.ndarray:
    """H = X X^T from token-major bf16 activations given as uint16 bit patterns (p x n)."""
    X = _c(X_bits, np.uint16)
    p, n = X.shape
    H = np.empty((n, n), np.float64)
    rc = _load().or_hessian_bf16(_p(X), p, n, _p(H))
    if rc:
        raise ValueError("or_hessian_bf16: invalid arguments")
    return H


def precondition(H, policy="adaptive", lam=0.0, tau=DEFAULT_TAU):
    """H' and delta (App. A Eqs. 23-24; Remark 1)."""
    H = _c(H, np.float64)
    n = H.shape[0]
    Hp = np.empty_like(H)
    d = np.empty(n, np.float64)
    rc = _load().or_precondition(_p(H), n, PRECOND[policy], float(lam), float(tau), _p(Hp), _p(d))
    if rc:
        raise ValueError("or_precondition: invalid arguments")
    return Hp, d


def cholesky(A):
    """L with A = L L^T (Eq. 9); raises NotPositiveDefinite(index)."""
    A = _c(A, np.float64)
    n = A.shape[0]
    L = np.empty_like(A)
    bad = _load().or_cholesky(_p(A), n, _p(L))
    if bad >= 0:
        raise NotPositiveDefinite(bad)
    return L


def init_codebook(W: np.ndarray, nbits: int) -> np.ndarray:
    """fp32 min-max grid T^0 (reading R-6 of P:218)."""
    W = _c(W, np.float32)
    m, n = W.shape
    T0 = np.empty((m, 1 << nbits), np.float32)
    _load().or_init_codebook(_p(W), m, n, 1 << nbits, _p(T0))
    return T0


def sstep(W, L, T):
    """Back-substitution S-step (Eqs. 15-22): returns (Q uint8, r fp64)."""
    W = _c(W, np.float64)
    L = _c(L, np.float64)
    T = _c(T, np.float64)
    m, n = W.shape
    Q = np.empty((m, n), np.uint8)
    R = np.empty((m, n), np.float64)
    _load().or_sstep(_p(W), _p(L), _p(T), m, n, T.shape[1], _p(Q), _p(R))
    return Q, R


def sstep_audit(W, L, T, Qg):
    """Teacher-forced audit of given codes Qg (parity rule P-3): (s_star, margin)."""
    W = _c(W, np.float64)
    L = _c(L, np.float64)
    T = _c(T, np.float64)
    Qg = _c(Qg, np.uint8)
    m, n = W.shape
    S = np.empty((m, n), np.uint8)
    M = np.empty((m, n), np.float64)
    _load().or_sstep_audit(_p(W), _p(L), _p(T), _p(Qg), m, n, T.shape[1], _p(S), _p(M))
    return S, M


def tstep(W, Q, H, nlev, empty_rule=0, Tprev=None, return_normal=False):
    """Closed-form T-step (Eq. 6) with raw H (reading R-4)."""
    W = _c(W, np.float64)
    Q = _c(Q, np.uint8)
    H = _c(H, np.float64)
    m, n = W.shape
    T = np.empty((m, nlev), np.float64)
    Tp = None if Tprev is None else _c(Tprev, np.float64)
    G = np.empty((m, nlev, nlev), np.float64) if return_normal else None
    b = np.empty((m, nlev), np.float64) if return_normal else None
    rc = _load().or_tstep(_p(W), _p(Q), _p(H), m, n, nlev, int(empty_rule), _p(Tp), _p(T), _p(G), _p(b))
    if rc:
        raise ValueError("or_tstep: invalid arguments")
    return (T, G, b) if return_normal else T


def objective(W, Q, T, H, per_row=False):
    """Eq. (1) via Eq. (8): sum_i e_i H e_i^T."""
    W = _c(W, np.float64)
    Q = _c(Q, np.uint8)
    T = _c(T, np.float64)
    H = _c(H, np.float64)
    m, n = W.shape
    pr = np.empty(m, np.float64)
    f = _load().or_objective(_p(W), _p(Q), _p(T), _p(H), m, n, T.shape[1], _p(pr))
    return (f, pr) if per_row else f


def quantize(W, H, nbits, iters, policy="adaptive", lam=0.0, tau=DEFAULT_TAU, T0=None,
             empty_rule=0, trace=False):
    """Algorithm 1 given H: returns (Q uint8, T fp64[, obj_trace])."""
    W = _c(W, np.float64)
    H = _c(H, np.float64)
    m, n = W.shape
    nlev = 1 << nbits
    Q = np.empty((m, n), np.uint8)
    T = np.empty((m, nlev), np.float64)
    tr = np.empty(iters, np.float64) if trace else None
    T0c = None if T0 is None else _c(T0, np.float32)
    rc = _load().or_quantize(_p(W), m, n, _p(H), nbits, iters, PRECOND[policy], float(lam), float(tau),
                             _p(T0c), int(empty_rule), _p(Q), _p(T), _p(tr))
    if rc == -2:
        raise ValueError("or_quantize: invalid arguments")
    if rc >= 0:
        raise NotPositiveDefinite(rc)
    return (Q, T, tr) if trace else (Q, T)


# --------------------------------------------------------------------------- NEXT-1
def pack(Q, nbits: int) -> np.ndarray:
    """Per-row little-endian N-bit packing of the codes (Table 1); rows padded
    to whole bytes.  Raises ValueError naming the first code >= 2^N."""
    lib = _load()
    Q = np.ascontiguousarray(Q, dtype=np.uint8)
    m, n = Q.shape
    out = np.zeros((m, (n * nbits + 7) // 8), dtype=np.uint8)
    bad = lib.or_pack(Q.ctypes.data, m, n, nbits, out.ctypes.data)
    if bad >= 0:
        raise ValueError(f"code {int(Q.flat[bad])} at flat index {bad} >= 2^{nbits}")
    return out


def unpack(Pk, m: int, n: int, nbits: int) -> np.ndarray:
    lib = _load()
    Pk = np.ascontiguousarray(Pk, dtype=np.uint8)
    Q = np.zeros((m, n), dtype=np.uint8)
    lib.or_unpack(Pk.ctypes.data, m, n, nbits, Q.ctypes.data)
    return Q


def lut_gemm(Pk, T16, X16, m: int, n: int, nbits: int) -> np.ndarray:
    """Y (p x m, fp64) = X W~^T, W~_ij = T16[i][Q_ij] (Fig. 1a right).
    T16 (m x 2^N) and X16 (p x n) are float16 arrays."""
    lib = _load()
    Pk = np.ascontiguousarray(Pk, dtype=np.uint8)
    T16 = np.ascontiguousarray(T16, dtype=np.float16)
    X16 = np.ascontiguousarray(X16, dtype=np.float16)
    p = X16.shape[0]
    Y = np.zeros((p, m), dtype=np.float64)
    lib.or_lut_gemm(Pk.ctypes.data, T16.view(np.uint16).ctypes.data, X16.view(np.uint16).ctypes.data,
                    m, n, p, nbits, Y.ctypes.data)
    return Y


STORAGE = {"fp16": 0, "uniform": 1, "lut": 2}


def storage_bytes(m: int, n: int, nbits: int, scheme: str) -> float:
    """Table 1: fp16 2mn; uniform mnN/8 + 4m; LUT mnN/8 + 2*2^N*m."""
    return _load().or_storage_bytes(m, n, nbits, STORAGE[scheme])


# --------------------------------------------------------------------------- NEXT-2
def outlier_indices(n: int, r: float):
    """(upper, lower): Algorithm 2's cutoff indices into the sorted row, 0-based."""
    up, lo = ctypes.c_int64(), ctypes.c_int64()
    _load().or_outlier_indices(n, r, ctypes.byref(up), ctypes.byref(lo))
    return up.value, lo.value


def outlier_split(W, r: float):
    """Algorithm 2: returns (mask uint8, W_dense fp32, c_lower, c_upper) per row."""
    lib = _load()
    W = np.ascontiguousarray(W, dtype=np.float32)
    m, n = W.shape
    M = np.zeros((m, n), np.uint8)
    Wd = np.zeros((m, n), np.float32)
    clo = np.zeros(m, np.float32)
    chi = np.zeros(m, np.float32)
    lib.or_outlier_split(W.ctypes.data, m, n, r, M.ctypes.data, Wd.ctypes.data, clo.ctypes.data, chi.ctypes.data)
    return M, Wd, clo, chi


def csr_of(W, M):
    """CSR (offsets int64, columns int32 ascending, values fp32) of W o M (the mask's entries)."""
    m, n = W.shape
    counts = M.sum(axis=1).astype(np.int64)
    off = np.zeros(m + 1, np.int64)
    off[1:] = np.cumsum(counts)
    rows, cols = np.nonzero(M)
    return off, cols.astype(np.int32), W[rows, cols].astype(np.float32)


def sparse_matmul(off, col, val, m: int, n: int, X) -> np.ndarray:
    """Y (p x m, fp64) = X W_sparse^T (the sparse path of GANQ*)."""
    lib = _load()
    off = np.ascontiguousarray(off, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float32)
    X = np.ascontiguousarray(X, np.float64)
    p = X.shape[0]
    Y = np.zeros((p, m), np.float64)
    lib.or_sparse_matmul(off.ctypes.data, col.ctypes.data, val.ctypes.data, m, n, X.ctypes.data, p, Y.ctypes.data)
    return Y


# --------------------------------------------------------------------------- NEXT-4
def kmeans_codebook(W, nbits: int, iters: int) -> np.ndarray:
    """Per-row 1-D Lloyd from the min-max grid (reading R-24): fp32 m x 2^N."""
    lib = _load()
    W = np.ascontiguousarray(W, dtype=np.float32)
    m, n = W.shape
    T = np.zeros((m, 1 << nbits), np.float32)
    lib.or_kmeans_codebook(W.ctypes.data, m, n, 1 << nbits, iters, T.ctypes.data)
    return T
