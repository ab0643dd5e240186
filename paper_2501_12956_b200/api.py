"""Python binding of the GANQ C ABI (include/ganq.h), same names, torch tensors in and out.

Argument marshalling only.  PyTorch provides device memory and the current CUDA stream;
every step of the method runs in libganq.so's sm_100a kernels.  Inputs must already be
CUDA tensors of the documented dtype -- there is no CPU path and no silent conversion of
device placement.
"""
from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _lib

__all__ = ["hessian", "hessian_partials", "hessian_fixed", "hessian_finalize", "hessian_fixed_size",
           "quantize_layer", "objective", "tstep", "factor", "workspace_size",
           "objective_workspace_size", "version", "pack_codes", "codebook_f16", "lut_gemm", "outlier_split",
           "sparse_gemm_add"]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@contextlib.contextmanager
def _on(dev, stream=None):
    """Run a call on dev: that device current, and `stream` (default: dev's current stream) the
    current stream, so outputs and workspace are allocated on the stream the kernels run on."""
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    if s.device != dev:
        raise ValueError(f"stream is on {s.device}, tensors on {dev}")
    with torch.cuda.device(dev), torch.cuda.stream(s):
        yield s


def _need(t, dtype, ndim, name, shape=None, device=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the GANQ path has no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}; every tensor of the call must be on {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


_ws_cache: dict = {}


def _workspace(nbytes: int, device, stream) -> torch.Tensor:
    """Scratch for one call, cached per (device, stream).  It is allocated while `stream` is the
    current stream, so the caching allocator orders its reuse after the kernels queued on that
    stream; calls on different streams never share a buffer."""
    key = (device.index, stream.cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        _ws_cache.pop(key, None)  # freed in stream order on `stream`
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def version() -> str:
    return _lib.load().ganq_version().decode()


def workspace_size(m: int, n: int, n_bits: int) -> int:
    return int(_lib.load().ganq_workspace_size(m, n, n_bits))


def objective_workspace_size(m: int, n: int) -> int:
    return int(_lib.load().ganq_objective_workspace_size(m, n))


def hessian(X: torch.Tensor, H: torch.Tensor | None = None, accumulate: bool = False, stream=None):
    """H = X X^T from token-major bf16 activations X (p x n); returns fp64 n x n."""
    _need(X, torch.bfloat16, 2, "X")
    p, n = X.shape
    dev = X.device
    with _on(dev, stream) as s:
        if H is None:
            if accumulate:
                raise ValueError("accumulate=True needs an existing H")
            H = torch.empty((n, n), dtype=torch.float64, device=dev)
        _need(H, torch.float64, 2, "H", shape=(n, n), device=dev)
        lib = _lib.load()
        _lib.check(lib.ganq_hessian(_ptr(X), p, n, _ptr(H), int(bool(accumulate)), _stream(s)))
    return H


SUPERCHUNK = 32768  # == GANQ_HESSIAN_SUPERCHUNK (include/ganq.h): token shards must be multiples


def hessian_fixed_size(n: int) -> int:
    """int64 entries of the fixed-point Hessian accumulator for n channels."""
    return int(_lib.load().ganq_hessian_fixed_size(n)) // 8


def hessian_partials(X: torch.Tensor, P: torch.Tensor | None = None, E: torch.Tensor | None = None, stream=None):
    """(P, E): the fp32 super-chunk partial sums of X X^T (ganq_hessian_partials, tile layout) and
    the int32 [n] grid exponents of its super-chunks' diagonals (include/ganq.h, reading R-12)."""
    _need(X, torch.bfloat16, 2, "X")
    p, n = X.shape
    dev = X.device
    lib = _lib.load()
    with _on(dev, stream) as s:
        if P is None:
            P = torch.empty(int(lib.ganq_hessian_partials_size(p, n)) // 4, dtype=torch.float32, device=dev)
        if E is None:
            E = torch.empty(n, dtype=torch.int32, device=dev)
        _need(P, torch.float32, 1, "P", shape=(int(lib.ganq_hessian_partials_size(p, n)) // 4,), device=dev)
        _need(E, torch.int32, 1, "E", shape=(n,), device=dev)
        _lib.check(lib.ganq_hessian_partials(_ptr(X), p, n, _ptr(P), _ptr(E), _stream(s)))
    return P, E


def hessian_fixed(P: torch.Tensor, p: int, E: torch.Tensor, Hfix: torch.Tensor | None = None,
                  accumulate: bool = False, stream=None):
    """The exact int64 sum of the partials of p tokens on the grid of E (ganq_hessian_fixed): tile
    layout; shards add exactly (torch / NCCL int64 SUM, any order)."""
    _need(E, torch.int32, 1, "E")
    n = E.shape[0]
    dev = E.device
    lib = _lib.load()
    _need(P, torch.float32, 1, "P", shape=(int(lib.ganq_hessian_partials_size(p, n)) // 4,), device=dev)
    with _on(dev, stream) as s:
        if Hfix is None:
            if accumulate:
                raise ValueError("accumulate=True needs an existing Hfix")
            Hfix = torch.empty(hessian_fixed_size(n), dtype=torch.int64, device=dev)
        _need(Hfix, torch.int64, 1, "Hfix", shape=(hessian_fixed_size(n),), device=dev)
        _lib.check(lib.ganq_hessian_fixed(_ptr(P), int(p), n, _ptr(E), _ptr(Hfix), int(bool(accumulate)), _stream(s)))
    return Hfix


def hessian_finalize(Hfix: torch.Tensor, E: torch.Tensor, H: torch.Tensor | None = None, accumulate: bool = False,
                     stream=None):
    """fp64 n x n symmetric H from the fixed-point accumulator (ganq_hessian_finalize)."""
    _need(E, torch.int32, 1, "E")
    n = E.shape[0]
    dev = E.device
    _need(Hfix, torch.int64, 1, "Hfix", shape=(hessian_fixed_size(n),), device=dev)
    with _on(dev, stream) as s:
        if H is None:
            if accumulate:
                raise ValueError("accumulate=True needs an existing H")
            H = torch.empty((n, n), dtype=torch.float64, device=dev)
        _need(H, torch.float64, 2, "H", shape=(n, n), device=dev)
        _lib.check(_lib.load().ganq_hessian_finalize(_ptr(Hfix), _ptr(E), n, _ptr(H), int(bool(accumulate)),
                                                     _stream(s)))
    return H


def _opts(precond, lam, tau, T0, empty_level_rule, trace_buf):
    o = _lib.Opts()
    if precond not in _lib.PRECOND:
        raise ValueError(f"unknown precond {precond!r}")
    o.precond = _lib.PRECOND[precond]
    o.empty_level_rule = int(empty_level_rule)
    o.lam = float(lam)
    o.tau = float(tau)
    o.T0 = None if T0 is None else T0.data_ptr()
    o.obj_trace = trace_buf
    return o


def quantize_layer(W: torch.Tensor, H: torch.Tensor, n_bits: int, iters: int = 10, *,
                   precond: str = "adaptive", lam: float = 0.0, tau: float = 1e-7,
                   T0: torch.Tensor | None = None, empty_level_rule: int = 0, trace: bool = False,
                   Q: torch.Tensor | None = None, T: torch.Tensor | None = None, stream=None,
                   init: str = "grid", kmeans_iters: int = 25):
    """Algorithm 1 given H: returns (Q uint8 m x n, T fp32 m x 2^N[, obj_trace]).

    precond: "adaptive" (App. A, default), "fixed_lambda" (H + lam I, Remark 1), "none", or
    "auto" (none, falling back to adaptive on a non-positive pivot).
    init (when T0 is None): "grid" (fp32 min-max grid, R-6) or "kmeans" (kmeans_codebook, R-24)."""
    if T0 is None and init == "kmeans":
        T0 = kmeans_codebook(W, n_bits, kmeans_iters, stream=stream)
    elif init not in ("grid", "kmeans"):
        raise ValueError(f"init must be 'grid' or 'kmeans', got {init!r}")
    if precond == "auto":
        # NEXT-4 "on failure only": no preconditioning unless the factor hits a non-positive
        # pivot, then the adaptive shift of App. A
        try:
            return quantize_layer(W, H, n_bits, iters, precond="none", lam=lam, tau=tau, T0=T0,
                                  empty_level_rule=empty_level_rule, trace=trace, Q=Q, T=T, stream=stream)
        except _lib.NotPositiveDefinite:
            return quantize_layer(W, H, n_bits, iters, precond="adaptive", lam=lam, tau=tau, T0=T0,
                                  empty_level_rule=empty_level_rule, trace=trace, Q=Q, T=T, stream=stream)
    _need(W, torch.float32, 2, "W")
    m, n = W.shape
    dev = W.device
    nlev = 1 << int(n_bits)
    _need(H, torch.float64, 2, "H", shape=(n, n), device=dev)
    if T0 is not None:
        _need(T0, torch.float32, 2, "T0", shape=(m, nlev), device=dev)
    with _on(dev, stream) as s:
        if Q is None:
            Q = torch.empty((m, n), dtype=torch.uint8, device=dev)
        if T is None:
            T = torch.empty((m, nlev), dtype=torch.float32, device=dev)
        _need(Q, torch.uint8, 2, "Q", shape=(m, n), device=dev)
        _need(T, torch.float32, 2, "T", shape=(m, nlev), device=dev)
        lib = _lib.load()
        nbytes = int(lib.ganq_workspace_size(m, n, int(n_bits)))
        ws = _workspace(nbytes, dev, s)
        tr = (ctypes.c_double * int(iters))() if trace else None
        o = _opts(precond, lam, tau, T0, empty_level_rule,
                  ctypes.cast(tr, ctypes.POINTER(ctypes.c_double)) if trace else None)
        _lib.check(lib.ganq_quantize_layer(_ptr(W), m, n, _ptr(H), int(n_bits), int(iters), ctypes.byref(o),
                                           _ptr(Q), _ptr(T), _ptr(ws), ws.numel(), _stream(s)))
    if trace:
        return Q, T, [float(x) for x in tr]
    return Q, T


def quantize_stacked(Ws, H: torch.Tensor, n_bits: int, iters: int = 10, *, T0=None, trace: bool = False,
                     stream=None, **kw):
    """Linears that read the same input (q/k/v, gate/up) share H = X X^T and so
    its factor L: their weights are stacked row-wise into one problem, solved once (one
    preconditioning + factorisation, one W H GEMM, one launch sequence per iteration) and split
    back.  Eq. (4) decomposes the objective over rows and every GPU kernel is row-local
    (per-row scales, row groups), so each block's (Q, T) equals a separate quantize_layer call
    bit for bit (tests/test_gpu_pipeline.py).  Returns [(Q_i, T_i)] as views of the stacked
    outputs (plus the stacked objective trace when trace=True)."""
    Ws = list(Ws)
    if not Ws:
        raise ValueError("quantize_stacked: need at least one weight matrix")
    n = H.shape[0]
    for k, W in enumerate(Ws):
        _need(W, torch.float32, 2, f"Ws[{k}]")
        if W.shape[1] != n or W.device != Ws[0].device:
            raise ValueError(f"quantize_stacked: Ws[{k}] is {tuple(W.shape)} on {W.device}; need (*, {n}) on "
                             f"{Ws[0].device}")
    rows = [W.shape[0] for W in Ws]
    W = Ws[0] if len(Ws) == 1 else torch.cat(Ws, 0)
    if T0 is not None and not isinstance(T0, torch.Tensor):
        T0 = torch.cat(list(T0), 0)
    res = quantize_layer(W, H, n_bits, iters, T0=T0, trace=trace, stream=stream, **kw)
    out = list(zip(res[0].split(rows, 0), res[1].split(rows, 0)))
    return (out, res[2]) if trace else out


def objective(W, Q, T, H, per_row: bool = False, stream=None):
    """Eq. (1) via Eq. (8) on raw H; returns a Python float (and the fp64 per-row tensor)."""
    _need(W, torch.float32, 2, "W")
    m, n = W.shape
    dev = W.device
    _need(Q, torch.uint8, 2, "Q", shape=(m, n), device=dev)
    _need(T, torch.float32, 2, "T", device=dev)
    nlev = int(T.shape[1])
    if T.shape[0] != m or nlev < 2 or nlev & (nlev - 1) or nlev > 256:
        raise ValueError(f"T must be m x 2^N (m = {m}, 1 <= N <= 8), got {tuple(T.shape)}")
    _need(H, torch.float64, 2, "H", shape=(n, n), device=dev)
    n_bits = nlev.bit_length() - 1
    with _on(dev, stream) as s:
        lib = _lib.load()
        ws = _workspace(int(lib.ganq_objective_workspace_size(m, n)), dev, s)
        out = ctypes.c_double(0.0)
        pr = torch.empty(m, dtype=torch.float64, device=dev) if per_row else None
        _lib.check(lib.ganq_objective(_ptr(W), _ptr(Q), _ptr(T), _ptr(H), m, n, n_bits, ctypes.byref(out),
                                      _ptr(pr), _ptr(ws), ws.numel(), _stream(s)))
    return (out.value, pr) if per_row else out.value


def tstep(W, Q, H, n_bits: int, empty_level_rule: int = 0, Tprev=None, stream=None):
    """T-update alone (Eq. 6) for given codes Q; returns fp32 m x 2^N."""
    _need(W, torch.float32, 2, "W")
    m, n = W.shape
    dev = W.device
    nlev = 1 << int(n_bits)
    _need(Q, torch.uint8, 2, "Q", shape=(m, n), device=dev)
    _need(H, torch.float64, 2, "H", shape=(n, n), device=dev)
    if Tprev is not None:
        _need(Tprev, torch.float32, 2, "Tprev", shape=(m, nlev), device=dev)
    with _on(dev, stream) as s:
        T = torch.empty((m, nlev), dtype=torch.float32, device=dev)
        lib = _lib.load()
        ws = _workspace(int(lib.ganq_workspace_size(m, n, n_bits)), dev, s)
        _lib.check(lib.ganq_tstep(_ptr(W), _ptr(Q), _ptr(H), m, n, int(n_bits), int(empty_level_rule),
                                  _ptr(Tprev), _ptr(T), _ptr(ws), ws.numel(), _stream(s)))
    return T


def factor(H, precond: str = "adaptive", lam: float = 0.0, tau: float = 1e-7, stream=None):
    """(L, delta): Cholesky of the preconditioned H (App. A / Remark 1 / Eq. 9)."""
    _need(H, torch.float64, 2, "H")
    n = H.shape[0]
    dev = H.device
    _need(H, torch.float64, 2, "H", shape=(n, n))
    with _on(dev, stream) as s:
        L = torch.empty_like(H)
        delta = torch.empty(n, dtype=torch.float64, device=dev)
        lib = _lib.load()
        ws = _workspace(int(lib.ganq_workspace_size(1, n, 1)), dev, s)
        o = _opts(precond, lam, tau, None, 0, None)
        _lib.check(lib.ganq_factor(_ptr(H), n, ctypes.byref(o), _ptr(L), _ptr(delta), _ptr(ws), ws.numel(),
                                   _stream(s)))
    return L, delta


# --------------------------------------------------------------------------- NEXT-1
def pack_codes(Q, n_bits: int, stream=None, check: bool = True):
    """Per-row little-endian N-bit packing of Q (Table 1 storage) -> uint8 m x ceil(nN/8).

    check=True verifies on the device that every code is < 2^N (the kernel stores only the low
    N bits of a code) and raises ValueError otherwise."""
    _need(Q, torch.uint8, 2, "Q")
    m, n = Q.shape
    with _on(Q.device, stream) as s:
        if check and int(Q.max()) >= (1 << n_bits):
            raise ValueError(f"codes must be < 2^{n_bits}")
        lib = _lib.load()
        P = torch.empty((m, int(lib.ganq_packed_row_bytes(n, int(n_bits)))), dtype=torch.uint8, device=Q.device)
        _lib.check(lib.ganq_pack_codes(_ptr(Q), m, n, int(n_bits), _ptr(P), _stream(s)))
    return P


def kmeans_codebook(W, n_bits: int, iters: int = 25, T=None, stream=None):
    """T^0 = per-row 1-D Lloyd k-means of W from the min-max grid (NEXT-4, reading R-24):
    fp32 m x 2^N on W's device."""
    _need(W, torch.float32, 2, "W")
    m, n = W.shape
    with _on(W.device, stream) as s:
        if T is None:
            T = torch.empty((m, 1 << int(n_bits)), dtype=torch.float32, device=W.device)
        _need(T, torch.float32, 2, "T", shape=(m, 1 << int(n_bits)), device=W.device)
        _lib.check(_lib.load().ganq_kmeans_codebook(_ptr(W), m, n, int(n_bits), int(iters), _ptr(T), _stream(s)))
    return T


def _nbits_of(nl: int, name: str) -> int:
    if nl < 2 or nl & (nl - 1) or nl > 256:
        raise ValueError(f"{name} must have 2^N columns (1 <= N <= 8), got {nl}")
    return int(nl).bit_length() - 1


def codebook_f16(T, stream=None):
    """fp32 codebook (m x 2^N) -> fp16 (round to nearest even), the stored form of Table 1."""
    _need(T, torch.float32, 2, "T")
    m, nl = T.shape
    n_bits = _nbits_of(nl, "T")
    with _on(T.device, stream) as s:
        T16 = torch.empty((m, nl), dtype=torch.float16, device=T.device)
        _lib.check(_lib.load().ganq_codebook_f16(_ptr(T), m, n_bits, _ptr(T16), _stream(s)))
    return T16


def lut_gemm(P, T16, X, n: int, Y=None, stream=None):
    """Y (p x m, fp32) = X W~^T for W~_ij = T16[i][Q_ij] decoded from the packed codes
    (Fig. 1a right).  X: p x n fp16 (token-major)."""
    _need(X, torch.float16, 2, "X")
    dev = X.device
    _need(T16, torch.float16, 2, "T16", device=dev)
    m, nl = T16.shape
    n_bits = _nbits_of(nl, "T16")
    p = X.shape[0]
    if X.shape[1] != n:
        raise ValueError("X must be p x n")
    _need(P, torch.uint8, 2, "packed", shape=(m, (n * n_bits + 7) // 8), device=dev)
    with _on(dev, stream) as s:
        if Y is None:
            Y = torch.empty((p, m), dtype=torch.float32, device=dev)
        _need(Y, torch.float32, 2, "Y", shape=(p, m), device=dev)
        _lib.check(_lib.load().ganq_lut_gemm(_ptr(P), _ptr(T16), _ptr(X), m, n, p, n_bits, _ptr(Y), _stream(s)))
    return Y


# --------------------------------------------------------------------------- NEXT-2
def outlier_split(W, r: float, stream=None):
    """GANQ* decomposition, Algorithm 2: returns (W_dense, csr, cutoffs) with
    csr = (row_offsets int64 m+1, col_idx int32, values fp32) of W_sparse and cutoffs =
    (c_lower, c_upper) per row."""
    _need(W, torch.float32, 2, "W")
    m, n = W.shape
    dev = W.device
    with _on(dev, stream) as s:
        Wd = torch.empty_like(W)
        clo = torch.empty(m, dtype=torch.float32, device=dev)
        chi = torch.empty(m, dtype=torch.float32, device=dev)
        off = torch.empty(m + 1, dtype=torch.int64, device=dev)
        nnz = ctypes.c_int64(0)
        lib = _lib.load()
        _lib.check(lib.ganq_outlier_split(_ptr(W), m, n, float(r), _ptr(Wd), _ptr(clo), _ptr(chi), _ptr(off),
                                          ctypes.byref(nnz), _stream(s)))
        col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)[: nnz.value]
        val = torch.empty(max(nnz.value, 1), dtype=torch.float32, device=dev)[: nnz.value]
        _lib.check(lib.ganq_outlier_csr(_ptr(W), m, n, _ptr(clo), _ptr(chi), _ptr(off), _ptr(col), _ptr(val),
                                        _stream(s)))
    return Wd, (off, col, val), (clo, chi)


def sparse_gemm_add(csr, X, Y, stream=None):
    """Y (p x m fp32) += X W_sparse^T for the CSR of outlier_split; X: p x n fp16."""
    off, col, val = csr
    _need(X, torch.float16, 2, "X")
    dev = X.device
    m = off.numel() - 1
    p, n = X.shape
    _need(Y, torch.float32, 2, "Y", shape=(p, m), device=dev)
    for t, nm in ((off, "row_offsets"), (col, "col_idx"), (val, "values")):
        if not t.is_cuda or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous CUDA tensor on {dev}")
    with _on(dev, stream) as s:
        _lib.check(_lib.load().ganq_sparse_gemm_add(_ptr(off), _ptr(col), _ptr(val), m, n, _ptr(X), p, _ptr(Y),
                                                    _stream(s)))
    return Y
