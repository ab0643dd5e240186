"""Independent formulations used to PIN the oracle (never used by it, never by the CUDA path).

Each routine restates a textbook special case or an alternative derivation of
a GANQ step with numpy, sharing no arithmetic with oracle/ganq_oracle.c:

* ``gptq_reverse_sstep`` -- the S-step with T fixed, as reverse-column-order
  OBS/GPTQ sequential rounding with compensation through the inverse of the
  leading block of H' (no Cholesky factor at all).  Equivalent to Eq. 22
   because x_F = w_F + H_FF^{-1} H_FR d_R has last component
  w_j + (1/L_jj) sum_{u>j} L_uj d_u for H = L L^T.
* ``bruteforce_s`` / ``bruteforce_solver`` -- exhaustive search over all
  assignments ("brute-force search over all combinations").
* ``lloyd_1d`` -- per-row 1-D Lloyd k-means (GANQ with H = I, P:139-142 with
  S H S^T diagonal = cluster counts).
* ``xform_objective`` -- Eq. (1) evaluated through X directly.
* ``tstep_lstsq`` -- the T-subproblem (Eq. 4) solved as an ordinary
  least-squares problem on the p x 2^N design matrix (numpy lstsq, min-norm).
"""
from __future__ import annotations

import itertools

import numpy as np


def nearest_first(z, t):
    d = np.abs(z - np.asarray(t))
    return int(np.flatnonzero(d == d.min())[0])


def gptq_reverse_sstep(W, Hp, T):
    W = np.asarray(W, np.float64)
    m, n = W.shape
    Q = np.zeros((m, n), np.uint8)
    for i in range(m):
        w = W[i].copy()
        for j in range(n - 1, -1, -1):
            q = nearest_first(w[j], T[i])
            Q[i, j] = q
            if j == 0:
                break
            Finv = np.linalg.inv(Hp[: j + 1, : j + 1])
            err = (w[j] - T[i][q]) / Finv[j, j]
            w[:j] -= err * Finv[:j, j]
    return Q


def objective_H(W, Q, T, H):
    E = np.asarray(W, np.float64) - np.take_along_axis(np.asarray(T, np.float64), Q.astype(np.int64), axis=1)
    return float(np.einsum("ij,jk,ik->", E, H, E)), E


def xform_objective(W, Q, T, Xtok):
    """||W X - W~ X||_F^2 with X = Xtok^T (Xtok is p x n token-major)."""
    Wt = np.take_along_axis(np.asarray(T, np.float64), Q.astype(np.int64), axis=1)
    D = (np.asarray(W, np.float64) - Wt) @ np.asarray(Xtok, np.float64).T
    return float(np.sum(D * D))


def bruteforce_s(w, t, H):
    """min over all assignments q in {0..nlev-1}^n of (w - t[q]) H (w - t[q])^T, T fixed."""
    n = len(w)
    nlev = len(t)
    best = np.inf
    bestq = None
    for q in itertools.product(range(nlev), repeat=n):
        e = w - np.asarray(t)[list(q)]
        f = e @ H @ e
        if f < best:
            best, bestq = f, q
    return best, np.array(bestq)


def closed_form_t(w, q, H, nlev):
    S = np.zeros((nlev, len(w)))
    S[q, np.arange(len(w))] = 1.0
    G = S @ H @ S.T
    b = w @ H @ S.T
    return b @ np.linalg.pinv(G, rcond=1e-13, hermitian=True)


def bruteforce_solver(w, H, nlev):
    """Global optimum of Eq. (2) for one row: every assignment with its optimal T."""
    n = len(w)
    best = np.inf
    for q in itertools.product(range(nlev), repeat=n):
        q = np.array(q)
        t = closed_form_t(w, q, H, nlev)
        e = w - t[q]
        f = e @ H @ e
        if f < best:
            best = f
    return best


def lloyd_1d(W, T0, iters):
    """Per-row Lloyd: nearest level (first index on ties), cluster means, empty level -> 0."""
    W = np.asarray(W, np.float64)
    T = np.asarray(T0, np.float64).copy()
    m, n = W.shape
    nlev = T.shape[1]
    Q = np.zeros((m, n), np.uint8)
    for _ in range(iters):
        for i in range(m):
            d = np.abs(W[i][:, None] - T[i][None, :])
            Q[i] = np.argmin(d, axis=1)  # numpy argmin returns the first minimum
            Tn = np.zeros(nlev)
            for a in range(nlev):
                sel = Q[i] == a
                if sel.any():
                    Tn[a] = W[i][sel].mean()
            T[i] = Tn
    return Q, T


def tstep_lstsq(W, Q, Xtok, nlev):
    W = np.asarray(W, np.float64)
    X = np.asarray(Xtok, np.float64).T  # n x p
    m, n = W.shape
    T = np.zeros((m, nlev))
    for i in range(m):
        S = np.zeros((nlev, n))
        S[Q[i], np.arange(n)] = 1.0
        D = (S @ X).T  # p x nlev
        y = W[i] @ X
        T[i] = np.linalg.lstsq(D, y, rcond=None)[0]
    return T
