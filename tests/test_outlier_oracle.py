"""Pins of the NEXT-2 oracle (GANQ* outlier extraction, Algorithm 2) -- CPU only.

Checked against what the algorithm's definition fixes independently of its code: the rank
definition of an order statistic (exactly k row entries are smaller than the k-th smallest, for
distinct values), the closed-form per-row count, SPEC's hand example, exact reconstruction, and
a dense numpy matmul for the sparse product.
"""
import numpy as np
import pytest

import oracle
import synthetic


def test_indices_at_the_papers_ratio():
    # r = 0.5 %; n = 4096: p = 0.9975, floor(4085.76) = 4085, ceil(10.24) = 11
    assert oracle.outlier_indices(4096, 0.005) == (4085, 11)
    assert oracle.outlier_indices(11008, 0.005) == (10980, 28)


@pytest.mark.parametrize("m,n,r", [(6, 4096, 0.005), (5, 1000, 0.02), (3, 64, 0.1)])
def test_cutoffs_are_order_statistics_and_counts(m, n, r):
    rng = np.random.default_rng(n)
    W = rng.standard_t(3, size=(m, n)).astype(np.float32)  # heavy-tailed, distinct values
    up, lo = oracle.outlier_indices(n, r)
    M, Wd, clo, chi = oracle.outlier_split(W, r)
    for i in range(m):
        assert int((W[i] < chi[i]).sum()) == up      # rank definition of sorted[upper]
        assert int((W[i] < clo[i]).sum()) == lo      # ... and of sorted[lower]
        assert int(M[i].sum()) == (n - up) + (lo + 1)  # closed form for distinct values
    assert np.array_equal(Wd + W * M, W)               # exact reconstruction
    assert not Wd[M.astype(bool)].any()
    assert np.abs(Wd).max() < np.abs(W).max()


def test_spec_hand_example():
    # SPEC [OP] split_outliers example: row [-10, 0, 0, 0, 0, 10], r = 1/3 -> dense row all zeros,
    # sparse holds -10 and 10 (the zeros tie with the lower cutoff and are marked, value 0)
    W = np.array([[-10, 0, 0, 0, 0, 10]], np.float32)
    M, Wd, clo, chi = oracle.outlier_split(W, 1 / 3)
    assert not Wd.any()
    assert np.array_equal(W * M, W)
    assert chi[0] == 10 and clo[0] == 0


def test_synthetic_weights_outliers_are_the_planted_ones():
    # synthetic W = 0.02 N(0,1) with Bernoulli(0.005) entries x10 (P:242's 0.5 % ratio): the
    # extracted extremes are dominated by the planted outliers
    W = synthetic.make_weights(64, 4096, seed=3).numpy()
    M, Wd, _, _ = oracle.outlier_split(W, 0.005)
    assert np.abs(Wd).max() < np.abs(W[M.astype(bool)]).max()
    assert np.abs(Wd).max() <= 0.02 * 10


@pytest.mark.parametrize("p", [1, 3])
def test_sparse_matmul_matches_dense(p):
    rng = np.random.default_rng(p)
    m, n = 20, 300
    W = rng.normal(size=(m, n)).astype(np.float32)
    M, _, _, _ = oracle.outlier_split(W, 0.05)
    off, col, val = oracle.csr_of(W, M)
    X = rng.normal(size=(p, n))
    Y = oracle.sparse_matmul(off, col, val, m, n, X)
    np.testing.assert_allclose(Y, X @ (W * M).astype(np.float64).T, rtol=1e-12, atol=1e-12)
    Y0 = oracle.sparse_matmul(np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), m, n, X)
    assert not Y0.any()
