"""Pins for the oracle's k-means initial codebook (NEXT-4, reading R-24).

T0 = per-row 1-D Lloyd from the min-max grid.  Pinned to things other than itself:
  * iteration 0 is the min-max grid (or_init_codebook, pinned in test_oracle_pins);
  * each Lloyd iteration equals one GANQ iteration with H = I (the S-step reduces to nearest
    rounding, the T-step to the cluster mean, P:139-142 with H = I) -- a different code path
    of the oracle (or_sstep/or_tstep) with the "keep" empty rule;
  * Lloyd's descent property: the 1-D distortion never increases (textbook k-means);
  * closed form: rows with exactly 2^N well-separated value clusters converge to the cluster
    means; brute force: on tiny rows the converged 2-means result is the global optimum,
    found by enumerating every contiguous split of the sorted row.
"""
import numpy as np
import pytest

import synthetic


def _distortion(W, T):
    W = np.asarray(W, np.float64)
    T = np.asarray(T, np.float64)
    return np.sum(np.min((W[:, :, None] - T[:, None, :]) ** 2, axis=2), axis=1)


def test_kmeans_zero_iters_is_grid(oracle):
    W = synthetic.make_weights(6, 70, seed=3).numpy()
    np.testing.assert_array_equal(oracle.kmeans_codebook(W, 3, 0), oracle.init_codebook(W, 3))


@pytest.mark.parametrize("nbits", [2, 3, 4])
def test_kmeans_step_equals_ganq_identity_iteration(oracle, nbits):
    W = synthetic.make_weights(7, 96, seed=10 + nbits).numpy()
    n = W.shape[1]
    T = oracle.init_codebook(W, nbits)
    for k in range(1, 5):
        _, Tg = oracle.quantize(W.astype(np.float64), np.eye(n), nbits, 1, policy="none", T0=T,
                                empty_rule=1)
        T = Tg.astype(np.float32)
        np.testing.assert_array_equal(oracle.kmeans_codebook(W, nbits, k), T)


def test_kmeans_distortion_non_increasing(oracle):
    W = synthetic.make_weights(10, 256, seed=21).numpy()
    prev = _distortion(W, oracle.kmeans_codebook(W, 4, 0))
    for k in range(1, 9):
        cur = _distortion(W, oracle.kmeans_codebook(W, 4, k))
        assert np.all(cur <= prev * (1 + 1e-6) + 1e-12)  # fp32 rounding of the means only
        prev = cur


def test_kmeans_recovers_separated_clusters(oracle):
    rng = np.random.default_rng(4)
    centers = np.array([-3.0, -1.0, 0.5, 2.0], np.float64)
    W = np.empty((3, 400), np.float32)
    for i in range(3):
        lab = np.repeat(np.arange(4), 100)
        W[i] = (centers[lab] + 0.01 * rng.normal(size=400)).astype(np.float32)
        rng.shuffle(W[i])
    T = oracle.kmeans_codebook(W, 2, 10)
    for i in range(3):
        means = sorted(float(np.mean(W[i][np.abs(W[i] - c) < 0.5], dtype=np.float64)) for c in centers)
        np.testing.assert_allclose(np.sort(T[i]), means, rtol=0, atol=1e-6)


def test_kmeans_tiny_rows_global_optimum(oracle):
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(3, 9))
        w = np.sort(rng.normal(size=n)).astype(np.float32)
        w[: n // 2] -= 3.0  # two groups: Lloyd from the min-max grid reaches the global optimum
        W = w[None, :]
        T = oracle.kmeans_codebook(W, 1, 50)
        best = min(
            np.sum((w[:c] - w[:c].astype(np.float64).mean()) ** 2)
            + np.sum((w[c:] - w[c:].astype(np.float64).mean()) ** 2)
            for c in range(1, n)
        )
        assert _distortion(W, T)[0] == pytest.approx(best, rel=1e-5, abs=1e-9)


def test_kmeans_constant_and_empty_levels(oracle):
    W = np.zeros((2, 20), np.float32)
    W[0] = 0.25
    W[1, :10] = -1.0
    W[1, 10:] = 1.0
    T = oracle.kmeans_codebook(W, 3, 5)
    assert np.all(T[0] == np.float32(0.25))
    # row 1: only the end levels hold weights; interior levels keep their grid values
    g = oracle.init_codebook(W, 3)[1]
    assert T[1, 0] == -1.0 and T[1, 7] == 1.0
    np.testing.assert_array_equal(T[1, 1:7], g[1:7])


def _dp_optimal_sse(w, k):
    """Exact 1-D k-clustering by dynamic programming over the sorted row (clusters are contiguous)."""
    x = np.sort(np.asarray(w, np.float64))
    n = len(x)
    c1 = np.concatenate([[0.0], np.cumsum(x)])
    c2 = np.concatenate([[0.0], np.cumsum(x * x)])

    def sse(a, b):  # x[a:b]
        s = c1[b] - c1[a]
        return max(c2[b] - c2[a] - s * s / (b - a), 0.0)

    D = np.full((k + 1, n + 1), np.inf)
    D[0, 0] = 0.0
    for c in range(1, k + 1):
        for b in range(c, n + 1):
            D[c, b] = min(D[c - 1, a] + sse(a, b) for a in range(c - 1, b))
    return D[k, n]


def test_kmeans_spec_examples(oracle):
    T = oracle.kmeans_codebook(np.array([[0, 3, 3, 3]], np.float32), 1, 25)
    np.testing.assert_array_equal(np.sort(T[0]), [0.0, 3.0])
    T = oracle.kmeans_codebook(np.array([[0, 0, 10, 10]], np.float32), 1, 25)
    np.testing.assert_array_equal(np.sort(T[0]), [0.0, 10.0])


def test_kmeans_near_dp_optimum(oracle):
    """SPEC S:208's derived check: 25 Lloyd iterations within 5 % of the DP-optimal SSE (median)."""
    rng = np.random.default_rng(6)
    ratios = []
    for seed in range(60):
        w = rng.normal(size=48).astype(np.float32)
        T = oracle.kmeans_codebook(w[None, :], 2, 25)
        ratios.append(_distortion(w[None, :], T)[0] / _dp_optimal_sse(w, 4))
    assert min(ratios) >= 1 - 1e-6
    assert np.median(ratios) <= 1.05
