"""Parity helpers shared by the GPU tests (rules P-3..P-5 of DESIGN.md section 4).

Test infrastructure: calls the fp64 oracle (oracle/) and the C-ABI binding side by side; the
two never share arithmetic.  P:n = /root/reference/PAPER.md line n.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

NEAR_TIE = 1e-6  # north_star: codes bit-exact except near-ties within 1e-6 relative (P-3)


def audit(W, L, T, Q):
    """Teacher-forced audit of the GPU codes Q (rule P-3, Eq. 22 at P:207).

    The oracle recomputes every z_ij from the GIVEN codes of the columns u > j with the given
    codebook T and factor L.  Returns (n_mismatch, n_violations, max_margin_ratio, margins) where a
    violation is a mismatch whose margin |z - t_q| - |z - t_s*| exceeds 1e-6 max_s |T_is|."""
    Tn = np.asarray(T, np.float64)
    S, M = oracle.sstep_audit(np.asarray(W, np.float64), L, Tn, Q)
    scale = np.max(np.abs(Tn), axis=1, keepdims=True)
    mism = S != Q
    bad = mism & (M > NEAR_TIE * scale)
    ratio = M / np.maximum(scale, 1e-300)
    return int(mism.sum()), int(bad.sum()), float(ratio.max()) if ratio.size else 0.0, ratio


def gpu_trajectory(g, Wd, H, nbits, K, T0=None, **kw):
    """(T^0, [(Q^{k+1}, T^{k+1}) for k < K]) of the GPU solve, one iteration per call with the
    previous codebook injected as T0 (bitwise the same sequence as one K-iteration call: checked
    by the callers)."""
    if T0 is None:
        # T^0 = the fp32 min-max grid (R-6); the GPU's own grid is bitwise this one
        # (test_init_codebook_bitwise)
        T0 = torch.from_numpy(oracle.init_codebook(Wd.cpu().numpy(), nbits)).to(Wd.device)
    T0n = T0.cpu().numpy()
    traj = []
    Tk = T0
    while len(traj) < K:
        Qn, Tn = g.quantize_layer(Wd, H, nbits, 1, T0=Tk, **kw)
        traj.append((Qn.cpu().numpy(), Tn.cpu().numpy()))
        Tk = Tn
    return T0n, traj


def oracle_trajectory(W64, Hn, L, T0, nbits, K, empty_rule=0):
    """The oracle's Algorithm 1 loop, iteration by iteration in fp64 (the same calls
    or_quantize makes): [(Q^{k+1}, T^{k+1})]."""
    nlev = 1 << nbits
    Tk = np.asarray(T0, np.float64)
    out = []
    for _ in range(K):
        Qk, _ = oracle.sstep(W64, L, Tk)
        Tn = oracle.tstep(W64, Qk, Hn, nlev, empty_rule=empty_rule, Tprev=Tk)
        out.append((Qk, Tn))
        Tk = Tn
    return out


def classify_divergence(W64, L, T0, gtraj, otraj):
    """SURVEY P-5: for every row whose code trajectory differs, take the first iteration k and the
    highest column j (the back-substitution runs j = n-1 .. 0, Eq. 22) where the codes differ, and
    apply P-3 there with the GPU's codebook T^k and codes:
        margin_gpu = |z - t_{q_gpu}| - |z - t_{s*}| / max|T^k_i|  (z from the GPU's own state)
    and, for context, the same margin of the GPU's code under the ORACLE's T^k (its z, from the
    oracle's codebook; the codes of the columns u > j are the same on both sides):
        margin_or  = (|z_o - t^o_{q_gpu}| - |z_o - t^o_{q_or}|) / max|T^o_i|.
    Returns a list of dicts, one per diverged row."""
    K = len(gtraj)
    m = W64.shape[0]
    Tg_prev = [np.asarray(T0, np.float64)] + [np.asarray(t, np.float64) for _, t in gtraj[:-1]]
    To_prev = [np.asarray(T0, np.float64)] + [t for _, t in otraj[:-1]]
    rows = []
    for i in range(m):
        for k in range(K):
            d = np.nonzero(gtraj[k][0][i] != otraj[k][0][i])[0]
            if d.size:
                j = int(d.max())
                rows.append(dict(row=i, k=k, j=j))
                break
    for r in rows:
        i, k, j = r["row"], r["k"], r["j"]
        Qg = gtraj[k][0][i:i + 1]
        Tg = Tg_prev[k][i:i + 1]
        S, M = oracle.sstep_audit(W64[i:i + 1], L, Tg, Qg)
        r["margin_gpu"] = float(M[0, j] / np.max(np.abs(Tg)))
        r["gpu_is_argmin"] = bool(S[0, j] == Qg[0, j])
        To = To_prev[k][i:i + 1]
        So, Mo = oracle.sstep_audit(W64[i:i + 1], L, To, Qg)
        r["margin_or"] = float(Mo[0, j] / np.max(np.abs(To)))
        r["dT"] = float(np.max(np.abs(Tg - To)) / np.max(np.abs(To)))
    return rows


def to_dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
