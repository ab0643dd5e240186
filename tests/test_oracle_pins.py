"""Pins for the fp64 CPU oracle (CPU only).

The oracle (oracle/ganq_oracle.c) is checked against things other than itself:
hand-derived values (tests/golden/hand_examples.json, each cited), numpy
library routines (matmul, cholesky, inv, pinv, lstsq), closed forms (n = 1,
diagonal H, H = I -> 1-D Lloyd), brute-force enumeration, an
independent formulation of the S-step (reverse-order GPTQ/OBS with H'^{-1}),
and the invariants the paper's derivation implies (T-step optimality and
monotonicity, Eq. 8 = Eq. 1, Eq. 14 with the preconditioning offset).
"""
import json
import os

import numpy as np
import pytest
import torch

import synthetic
from tests import _pins

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))


def _spd(n, seed, diag=1.0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, 3 * n))
    return A @ A.T / (3 * n) + diag * np.eye(n)


def _bf16_tokens(p, n, seed):
    X = synthetic.make_activations(p, n, seed=seed)
    return synthetic.bf16_bits(X), synthetic.bf16_to_f64(X)


# ----------------------------------------------------------------------------- golden

def test_golden_cholesky(oracle):
    g = GOLD["cholesky_2x2"]
    np.testing.assert_array_equal(oracle.cholesky(np.array(g["A"])), np.array(g["L"]))
    g = GOLD["cholesky_not_pd"]
    with pytest.raises(oracle.NotPositiveDefinite) as ei:
        oracle.cholesky(np.array(g["A"]))
    assert ei.value.index == g["fail_index"]


def test_golden_hessian(oracle):
    for key in ("hessian_two_tokens", "hessian_identity"):
        g = GOLD[key]
        X = torch.tensor(g["X_tokens"], dtype=torch.float32).to(torch.bfloat16)
        H = oracle.hessian_bf16(synthetic.bf16_bits(X))
        np.testing.assert_array_equal(H, np.array(g["H"]))


def test_golden_precondition(oracle):
    g = GOLD["adaptive_identity"]
    Hp, d = oracle.precondition(np.array(g["H"]), "adaptive")
    np.testing.assert_allclose(d, g["delta"], rtol=1e-12)
    g = GOLD["adaptive_weak_dominance"]
    Hp, d = oracle.precondition(np.array(g["H"]), "adaptive")
    np.testing.assert_allclose(d, g["delta"], rtol=1e-12)
    L = oracle.cholesky(Hp)  # must succeed thanks to the jitter (reading R-3)
    np.testing.assert_allclose(L @ L.T, Hp, rtol=1e-12, atol=1e-12)
    # without the jitter the literal Eq. 23 matrix is singular: Cholesky fails at index 1
    Hp0, _ = oracle.precondition(np.array(g["H"]), "adaptive", tau=0.0)
    with pytest.raises(oracle.NotPositiveDefinite):
        oracle.cholesky(Hp0)
    g = GOLD["fixed_lambda_identity"]
    Hp, d = oracle.precondition(np.array(g["H"]), "fixed_lambda", lam=g["lambda"])
    np.testing.assert_array_equal(Hp, np.array(g["Hp"]))
    with pytest.raises(ValueError):
        oracle.precondition(np.eye(2), "fixed_lambda", lam=0.0)


def test_golden_single_level(oracle):
    g = GOLD["single_level_codebook"]
    T = oracle.tstep(np.array(g["W"]), np.array(g["Q"], np.uint8), np.array(g["H"]), nlev=4)
    assert T[0, 0] == pytest.approx(g["T0"], rel=1e-14)
    np.testing.assert_array_equal(T[0, 1:], 0.0)  # unused levels -> 0 (pinv, reading R-9)


def test_golden_n1_nearest(oracle):
    g = GOLD["n1_nearest"]
    W = np.array(g["W"])
    T = np.array(g["T"])
    Q, _ = oracle.sstep(W, np.array([[1.7]]), T)
    np.testing.assert_array_equal(Q, np.array(g["Q"], np.uint8))


# ----------------------------------------------------------------------------- Hessian / Cholesky

def test_hessian_matches_numpy(oracle):
    bits, Xd = _bf16_tokens(300, 40, seed=7)
    H = oracle.hessian_bf16(bits)
    ref = Xd.T @ Xd
    np.testing.assert_allclose(H, ref, rtol=1e-13, atol=1e-10)
    assert np.array_equal(H, H.T)


def test_cholesky_matches_numpy(oracle):
    for n, seed in ((1, 0), (7, 1), (64, 2)):
        A = _spd(n, seed)
        L = oracle.cholesky(A)
        np.testing.assert_allclose(L, np.linalg.cholesky(A), rtol=1e-11, atol=1e-13)
        assert np.all(np.triu(L, 1) == 0)


def test_adaptive_strictly_dominant(oracle):
    bits, Xd = _bf16_tokens(64, 48, seed=3)  # p < n: X X^T is singular
    bits = bits.copy()
    bits[:, 5] = 0  # a dead channel: H_55 = 0, so the 6th pivot is exactly 0
    H = oracle.hessian_bf16(bits)
    with pytest.raises(oracle.NotPositiveDefinite):
        oracle.cholesky(H)
    Hp, d = oracle.precondition(H, "adaptive")
    off = np.sum(np.abs(Hp), axis=1) - np.abs(np.diag(Hp))
    assert np.all(np.diag(Hp) > off)  # strict after the jitter
    rs = np.sum(np.abs(H), axis=1) - 2 * np.diag(H)
    np.testing.assert_allclose(d, np.maximum(rs, 1e-8) + 1e-7 * np.mean(np.diag(H)), rtol=1e-13)
    oracle.cholesky(Hp)  # succeeds
    Hl, _ = oracle.precondition(H, "fixed_lambda", lam=0.3)
    v = np.random.default_rng(0).normal(size=48)
    assert v @ Hl @ v >= 0.3 * v @ v * (1 - 1e-12)  # Remark 1 inequality


# ----------------------------------------------------------------------------- init codebook

def test_init_codebook_grid(oracle):
    W = synthetic.make_weights(5, 33, seed=11).numpy()
    W[2] = 0.125  # constant row -> all levels equal
    T0 = oracle.init_codebook(W, 3)
    assert T0.dtype == np.float32
    for i in range(5):
        mn, mx = np.float32(W[i].min()), np.float32(W[i].max())
        step = np.float32((mx - mn) / np.float32(7))
        exp = np.array([mn + np.float32(np.float32(s) * step) for s in range(8)], np.float32)
        np.testing.assert_array_equal(T0[i], exp)
    assert T0[0, 0] == W[0].min()
    assert np.all(T0[2] == np.float32(0.125))


# ----------------------------------------------------------------------------- S-step

def test_sstep_diagonal_is_nearest(oracle):
    rng = np.random.default_rng(5)
    W = rng.normal(size=(6, 17))
    T = np.sort(rng.normal(size=(6, 8)), axis=1)
    Hd = np.diag(rng.uniform(0.5, 2.0, size=17))
    L = np.sqrt(Hd)
    Q, R = oracle.sstep(W, L, T)
    ref = np.argmin(np.abs(W[:, :, None] - T[:, None, :]), axis=2)
    np.testing.assert_array_equal(Q, ref)
    np.testing.assert_allclose(R, W - np.take_along_axis(T, ref, 1), rtol=0, atol=0)


def test_sstep_term_by_term_argmin(oracle):
    """Each chosen code minimises the j-th squared term of Eq. (15) given later columns."""
    rng = np.random.default_rng(9)
    n, nlev = 10, 4
    W = rng.normal(size=(6, n))
    T = rng.normal(size=(6, nlev))
    L = np.linalg.cholesky(_spd(n, 4))
    Q, R = oracle.sstep(W, L, T)
    for i in range(6):
        for j in range(n):
            tail = sum(R[i, u] * L[u, j] for u in range(j + 1, n))
            terms = [(tail + (W[i, j] - T[i, s]) * L[j, j]) ** 2 for s in range(nlev)]
            assert terms[Q[i, j]] <= min(terms) * (1 + 1e-12) + 1e-300
            assert np.isclose(R[i, j], W[i, j] - T[i, Q[i, j]], rtol=0, atol=0)


def test_sstep_equals_reverse_gptq(oracle):
    """Independent formulation: reverse-order OBS/GPTQ with (H'_FF)^{-1}, no Cholesky factor."""
    W = synthetic.make_weights(12, 24, seed=21).numpy().astype(np.float64)
    bits, Xd = _bf16_tokens(96, 24, seed=22)
    H = oracle.hessian_bf16(bits)
    for pol, lam in (("adaptive", 0.0), ("fixed_lambda", 0.05 * np.mean(np.diag(H))), ("none", 0.0)):
        Hp, _ = oracle.precondition(H, pol, lam=lam)
        L = oracle.cholesky(Hp)
        T = oracle.init_codebook(W.astype(np.float32), 2).astype(np.float64)
        Q, _ = oracle.sstep(W, L, T)
        Qg = _pins.gptq_reverse_sstep(W, Hp, T)
        np.testing.assert_array_equal(Q, Qg)


def test_sstep_vs_bruteforce_fixed_T(oracle):
    """Greedy >= exhaustive min over all 4^n assignments (T fixed); equality for diagonal L."""
    rng = np.random.default_rng(31)
    n, nlev = 6, 4
    for trial in range(12):
        w = rng.normal(size=(1, n))
        t = np.sort(rng.normal(size=(1, nlev)), axis=1)
        Hp = _spd(n, 100 + trial, diag=0.3)
        L = np.linalg.cholesky(Hp)
        Q, _ = oracle.sstep(w, L, t)
        f_greedy, _ = _pins.objective_H(w, Q, t, Hp)
        f_best, _ = _pins.bruteforce_s(w[0], t[0], Hp)
        assert f_greedy >= f_best * (1 - 1e-12)
        Hd = np.diag(np.diag(Hp))
        Qd, _ = oracle.sstep(w, np.sqrt(Hd), t)
        fd, _ = _pins.objective_H(w, Qd, t, Hd)
        fbd, _ = _pins.bruteforce_s(w[0], t[0], Hd)
        assert fd == pytest.approx(fbd, rel=1e-12)


def test_sstep_audit_consistent(oracle):
    rng = np.random.default_rng(2)
    W = rng.normal(size=(5, 20))
    T = rng.normal(size=(5, 8))
    L = np.linalg.cholesky(_spd(20, 3))
    Q, _ = oracle.sstep(W, L, T)
    S, M = oracle.sstep_audit(W, L, T, Q)
    np.testing.assert_array_equal(S, Q)
    assert np.all(M == 0)
    Qbad = Q.copy()
    Qbad[2, 19] = (Qbad[2, 19] + 1) % 8
    S, M = oracle.sstep_audit(W, L, T, Qbad)
    assert M[2, 19] > 0 and S[2, 19] == Q[2, 19]


# ----------------------------------------------------------------------------- T-step

def test_tstep_normal_equations_and_lstsq(oracle):
    m, n, nlev = 7, 20, 8
    W = synthetic.make_weights(m, n, seed=41).numpy().astype(np.float64)
    bits, Xd = _bf16_tokens(120, n, seed=42)
    H = oracle.hessian_bf16(bits)
    rng = np.random.default_rng(43)
    Q = rng.integers(0, nlev, size=(m, n)).astype(np.uint8)
    Q[3] = rng.integers(0, 3, size=n)  # a row with 5 unused levels
    T, G, b = oracle.tstep(W, Q, H, nlev, return_normal=True)
    for i in range(m):
        S = np.zeros((nlev, n))
        S[Q[i], np.arange(n)] = 1
        np.testing.assert_allclose(G[i], S @ H @ S.T, rtol=1e-12, atol=1e-9)
        np.testing.assert_allclose(b[i], W[i] @ H @ S.T, rtol=1e-12, atol=1e-12)
        used = np.bincount(Q[i], minlength=nlev) > 0
        r = G[i] @ T[i] - b[i]
        assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b[i])
        assert np.all(T[i][~used] == 0)
    Tl = _pins.tstep_lstsq(W, Q, Xd, nlev)
    np.testing.assert_allclose(T, Tl, rtol=1e-7, atol=1e-9)
    # keep-previous empty rule (reading R-9 option 1)
    Tprev = np.full((m, nlev), 7.0)
    T1 = oracle.tstep(W, Q, H, nlev, empty_rule=1, Tprev=Tprev)
    used3 = np.bincount(Q[3], minlength=nlev) > 0
    np.testing.assert_array_equal(T1[3][~used3], 7.0)
    np.testing.assert_allclose(T1[3][used3], T[3][used3], rtol=1e-14)


def test_tstep_identity_is_cluster_mean(oracle):
    rng = np.random.default_rng(8)
    W = rng.normal(size=(4, 30))
    Q = rng.integers(0, 4, size=(4, 30)).astype(np.uint8)
    T = oracle.tstep(W, Q, np.eye(30), 4)
    for i in range(4):
        for a in range(4):
            sel = Q[i] == a
            exp = W[i][sel].mean() if sel.any() else 0.0
            assert T[i, a] == pytest.approx(exp, rel=1e-12, abs=1e-14)


def test_tstep_singular_uses_pinv(oracle):
    """Rank-deficient H (p < n, preconditioning off): T equals numpy's min-norm pinv solution."""
    m, n, nlev = 3, 12, 4
    bits, Xd = _bf16_tokens(2, n, seed=5)  # rank-2 H
    H = oracle.hessian_bf16(bits)
    rng = np.random.default_rng(6)
    W = rng.normal(size=(m, n))
    Q = rng.integers(0, nlev, size=(m, n)).astype(np.uint8)
    T = oracle.tstep(W, Q, H, nlev)
    for i in range(m):
        np.testing.assert_allclose(T[i], _pins.closed_form_t(W[i], Q[i], H, nlev), rtol=1e-6, atol=1e-9)


def test_init_codebook_closed_forms(oracle):
    """T^0 on rows whose grid is exactly representable (reading R-6; SPEC S:205's example): both
    endpoints are hit exactly and the step is (max - min) / (2^N - 1) -- a 2^N divisor or an
    off-by-one level count fails here."""
    cases = [([0.0, 1.0], 1, [0.0, 1.0]),
             ([-1.0, 2.0, 0.5], 2, [-1.0, 0.0, 1.0, 2.0]),
             ([3.0, -12.0, 0.0, 1.0], 2, [-12.0, -7.0, -2.0, 3.0]),
             ([0.0, 15.0, 7.0], 4, list(range(16))),
             ([2.0, 9.0], 3, [2.0 + s for s in range(8)])]
    for row, nb, exp in cases:
        T0 = oracle.init_codebook(np.array([row], np.float32), nb)
        np.testing.assert_array_equal(T0[0], np.array(exp, np.float32))
        assert T0[0, -1] == max(row) and T0[0, 0] == min(row)


@pytest.mark.parametrize("nlev,rank,seed", [(4, 1, 0), (4, 2, 1), (4, 3, 2), (8, 5, 3), (16, 9, 4), (16, 16, 5)])
def test_tstep_pinv_ranks(oracle, nlev, rank, seed):
    """The Moore-Penrose branch over ranks 1 .. 2^N of the normal matrix: H = X X^T with
    rank(H) = rank (p = rank tokens) and every level used, so G_i = S_i H S_i^T has that rank;
    T must equal numpy's pseudo-inverse solution b G^+ (SVD based, an independent routine) and
    lie in the row space of G (min-norm: orthogonal to its null space)."""
    n = 40
    rng = np.random.default_rng(seed)
    Xt = rng.normal(size=(rank, n))
    H = Xt.T @ Xt
    W = rng.normal(size=(3, n))
    Q = np.stack([rng.permutation(np.arange(n) % nlev) for _ in range(3)]).astype(np.uint8)
    T, G, b = oracle.tstep(W, Q, H, nlev, return_normal=True)
    for i in range(3):
        Gi = G[i]
        exp = b[i] @ np.linalg.pinv(Gi, rcond=1e-10, hermitian=True)
        scale = np.max(np.abs(exp))
        np.testing.assert_allclose(T[i], exp, rtol=0, atol=1e-8 * scale)
        w, V = np.linalg.eigh(Gi)
        null = V[:, w < 1e-9 * w.max()]
        assert np.all(np.abs(T[i] @ null) <= 1e-8 * scale)
        assert np.linalg.matrix_rank(Gi, tol=1e-9 * w.max()) == min(rank, nlev)


def test_tstep_monotone(oracle):
    m, n = 6, 32
    W = synthetic.make_weights(m, n, seed=51).numpy().astype(np.float64)
    bits, Xd = _bf16_tokens(200, n, seed=52)
    H = oracle.hessian_bf16(bits)
    Hp, _ = oracle.precondition(H, "adaptive")
    L = oracle.cholesky(Hp)
    T = oracle.init_codebook(W.astype(np.float32), 3).astype(np.float64)
    for _ in range(4):
        Q, _ = oracle.sstep(W, L, T)
        f_before = oracle.objective(W, Q, T, H)
        T = oracle.tstep(W, Q, H, 8)
        f_after = oracle.objective(W, Q, T, H)
        assert f_after <= f_before * (1 + 1e-12)


# ----------------------------------------------------------------------------- objective

def test_objective_identities(oracle):
    m, n, nlev = 5, 24, 8
    W = synthetic.make_weights(m, n, seed=61).numpy().astype(np.float64)
    bits, Xd = _bf16_tokens(150, n, seed=62)
    H = oracle.hessian_bf16(bits)
    rng = np.random.default_rng(63)
    Q = rng.integers(0, nlev, size=(m, n)).astype(np.uint8)
    T = rng.normal(scale=0.02, size=(m, nlev))
    f, pr = oracle.objective(W, Q, T, H, per_row=True)
    assert f == pytest.approx(_pins.xform_objective(W, Q, T, Xd), rel=1e-11)
    assert np.sum(pr) == pytest.approx(f, rel=1e-14)
    Hp, d = oracle.precondition(H, "adaptive")
    Lp = oracle.cholesky(Hp)
    _, E = _pins.objective_H(W, Q, T, H)
    lform = np.sum((E @ Lp) ** 2)
    assert lform == pytest.approx(f + np.sum(E * E * d[None, :]), rel=1e-10)  # Eq. 14 with H + Diag(delta)


# ----------------------------------------------------------------------------- whole solver

def test_solver_vs_global_optimum(oracle):
    """GANQ never beats the exhaustive global optimum of Eq. (2) (n = 6, N = 2)."""
    rng = np.random.default_rng(71)
    n = 6
    for trial in range(6):
        Xt = rng.normal(size=(40, n)).astype(np.float32)
        Xb = torch.from_numpy(Xt).to(torch.bfloat16)
        H = oracle.hessian_bf16(synthetic.bf16_bits(Xb))
        w = rng.normal(size=(1, n))
        Q, T = oracle.quantize(w, H, 2, 5, policy="none")
        f = oracle.objective(w, Q, T, H)
        fopt = _pins.bruteforce_solver(w[0], H, 4)
        assert f >= fopt * (1 - 1e-9)


def test_solver_exact_representability(oracle):
    W, A = synthetic.alphabet_weights(6, 40, 2, seed=9)
    bits, _ = _bf16_tokens(100, 40, seed=10)
    H = oracle.hessian_bf16(bits)
    Q, T, tr = oracle.quantize(W.astype(np.float64), H, 2, 3, T0=A, trace=True)
    idx = np.argmax(W[:, :, None] == A[:, None, :], axis=2)  # the alphabet index of every entry
    np.testing.assert_array_equal(Q, idx)
    np.testing.assert_allclose(T, A.astype(np.float64), rtol=1e-12, atol=0)
    assert tr[0] <= 1e-20 * np.sum(np.diag(H))


def test_solver_identity_is_lloyd(oracle):
    """H = I: S-step is nearest rounding, T-step the cluster mean -> per-row 1-D Lloyd from T^0."""
    W = synthetic.make_weights(8, 50, seed=81).numpy()
    T0 = oracle.init_codebook(W, 3)
    Q, T = oracle.quantize(W.astype(np.float64), np.eye(50), 3, 6, policy="none", T0=T0)
    Ql, Tl = _pins.lloyd_1d(W, T0, 6)
    np.testing.assert_array_equal(Q, Ql)
    np.testing.assert_allclose(T, Tl, rtol=1e-12, atol=1e-15)


def test_solver_row_independence_and_determinism(oracle):
    W = synthetic.make_weights(9, 40, seed=91).numpy().astype(np.float64)
    bits, _ = _bf16_tokens(160, 40, seed=92)
    H = oracle.hessian_bf16(bits)
    Q, T = oracle.quantize(W, H, 3, 4)
    Q2, T2 = oracle.quantize(W, H, 3, 4)
    np.testing.assert_array_equal(Q, Q2)
    np.testing.assert_array_equal(T, T2)
    for i in (0, 4, 8):
        Qi, Ti = oracle.quantize(W[i:i + 1], H, 3, 4)
        np.testing.assert_array_equal(Qi[0], Q[i])
        np.testing.assert_array_equal(Ti[0], T[i])


def test_solver_argument_errors(oracle):
    W = np.zeros((2, 3))
    H = np.eye(3)
    with pytest.raises(ValueError):
        oracle.quantize(W, H, 0, 3)
    with pytest.raises(ValueError):
        oracle.quantize(W, H, 2, 0)
    Hbad = np.array([[1.0, 2, 0], [2, 1, 0], [0, 0, 1]])
    with pytest.raises(oracle.NotPositiveDefinite) as ei:
        oracle.quantize(W, Hbad, 2, 1, policy="none")
    assert ei.value.index == 1


def test_solver_c1_runs_and_improves(oracle):
    """Config c1 (BASELINE.json configs[0]) end to end: objective far below the T^0 grid's."""
    c = synthetic.CONFIGS["c1"]
    W = synthetic.make_weights(c["m"], c["n"], seed=1000).numpy()
    X = synthetic.make_activations(c["p"], c["n"], seed=2000)
    H = oracle.hessian_bf16(synthetic.bf16_bits(X))
    T0 = oracle.init_codebook(W, c["nbits"])
    Hp, _ = oracle.precondition(H, "adaptive")
    Q0, _ = oracle.sstep(W.astype(np.float64), oracle.cholesky(Hp), T0.astype(np.float64))
    f_grid = oracle.objective(W.astype(np.float64), Q0, T0.astype(np.float64), H)
    Q, T, tr = oracle.quantize(W.astype(np.float64), H, c["nbits"], c["iters"], trace=True)
    assert tr[-1] < 0.5 * f_grid
    assert tr[-1] == pytest.approx(oracle.objective(W.astype(np.float64), Q, T, H), rel=1e-12)
