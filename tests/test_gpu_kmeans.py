"""NEXT-4 k-means T^0 (reading R-24) on the GPU vs the oracle, through the C ABI.

Bit-exact: assignments use fp64 distances of fp32 values (exact) with first-index ties on both
sides, and the per-level fp64 sums are exact for these rows, so the means and their fp32 rounding
agree bit for bit whatever the summation order (R-24).
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic
import paper_2501_12956_b200 as g

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _setup():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    oracle.build()


def _gpu(W, nbits, iters):
    T = g.kmeans_codebook(torch.from_numpy(W).to(DEV), nbits, iters)
    torch.cuda.synchronize()
    return T.cpu().numpy()


@pytest.mark.parametrize("nbits", [1, 2, 3, 4])
@pytest.mark.parametrize("iters", [0, 1, 25])
def test_kmeans_bitwise_small(nbits, iters):
    W = synthetic.make_weights(37, 300, seed=50 + nbits).numpy()  # ragged vs the 128-thread stride
    np.testing.assert_array_equal(_gpu(W, nbits, iters), oracle.kmeans_codebook(W, nbits, iters))


def test_kmeans_edge_rows():
    rng = np.random.default_rng(3)
    W = rng.normal(size=(6, 5)).astype(np.float32)
    W[0] = 0.5                      # constant row: every level equal, all weights on level 0
    W[1] = [0, 0, 10, 10, 10]       # two exact clusters, interior levels empty
    W[2] = [-1, 1, -1, 1, 0]        # exact ties between levels
    W[3] = [0.0, -0.0, 0.0, -0.0, 0.0]
    for nbits in (1, 2, 4):
        np.testing.assert_array_equal(_gpu(W, nbits, 25), oracle.kmeans_codebook(W, nbits, 25))
    W1 = rng.normal(size=(4, 1)).astype(np.float32)  # n = 1
    np.testing.assert_array_equal(_gpu(W1, 3, 5), oracle.kmeans_codebook(W1, 3, 5))


def test_kmeans_full_size_sampled_rows():
    """c2 shape (4096 x 4096), 25 iterations, in the launch the quantizer uses; rows are
    independent, so sampled rows are checked against the oracle one by one."""
    W = synthetic.make_weights(4096, 4096, seed=1001)
    T = g.kmeans_codebook(W.to(DEV), 4, 25).cpu().numpy()
    rows = np.random.default_rng(0).choice(4096, 48, replace=False)
    Wn = W.numpy()
    np.testing.assert_array_equal(T[rows], oracle.kmeans_codebook(Wn[rows], 4, 25))


def test_quantize_layer_kmeans_init_routes_T0():
    W = synthetic.make_weights(96, 256, seed=7).to(DEV)
    X = synthetic.make_activations(512, 256, seed=8).to(DEV)
    H = g.hessian(X)
    T0 = g.kmeans_codebook(W, 3, 25)
    Qa, Ta = g.quantize_layer(W, H, 3, 3, init="kmeans")
    Qb, Tb = g.quantize_layer(W, H, 3, 3, T0=T0)
    assert torch.equal(Qa, Qb) and torch.equal(Ta, Tb)


def test_kmeans_rejects_bad_args():
    W = torch.zeros((4, 8), device=DEV)
    with pytest.raises(g.GanqError):
        g.kmeans_codebook(W, 5, 3)
    with pytest.raises(g.GanqError):
        g.kmeans_codebook(W, 2, -1)


@pytest.mark.parametrize("nbits", [3, 4])
def test_quantize_from_kmeans_init_vs_oracle(nbits):
    """End to end from the k-means T0: the GPU's T0 equals the oracle's bit for bit, so both
    solvers start from the same codebook; the free-running solve then meets the same bars as
    the grid start (test_gpu_parity.py::test_free_running_end_to_end, R-13)."""
    m, n, p, K = 96, 512, 8192, 6
    W = synthetic.make_weights(m, n, seed=31)
    X = synthetic.make_activations(p, n, seed=32)
    H = g.hessian(X.to(DEV))
    T0o = oracle.kmeans_codebook(W.numpy(), nbits, 25)
    Qg, Tg = g.quantize_layer(W.to(DEV), H, nbits, K, init="kmeans", precond="none")
    Hn = H.cpu().numpy()
    Qo, To = oracle.quantize(W.numpy().astype(np.float64), Hn, nbits, K, policy="none", T0=T0o)
    fg, prg = g.objective(W.to(DEV), Qg, Tg, H, per_row=True)
    _, pro = oracle.objective(W.numpy().astype(np.float64), Qo, To, Hn, per_row=True)
    fo = float(np.sum(pro))
    prg = prg.cpu().numpy()
    same = np.all(Qg.cpu().numpy() == Qo, axis=1)
    assert np.all(np.abs(prg[same] - pro[same]) <= 1e-4 * pro[same])
    assert same.mean() >= 0.8
    assert abs(fg - fo) <= 1e-2 * fo, (fg, fo)
