"""NEXT-1 on the GPU vs the fp64 oracle, through the C ABI: packing, fp16 codebook, LUT mpGEMM.

Rules:
  packing: bit-exact (integer work);
  codebook: fp16 round-to-nearest-even, bit-exact against numpy's conversion;
  lut_gemm: |y - y_oracle| <= (8 ceil(n / 256) + 7) 2^-24 sum_j |W~_ij x_j| -- each lane adds
      its 8 ceil(n / 256) products in fp32 (fused multiply-add) in ascending j, then a 5-level
      butterfly; the bound is the first-order error of that summation tree (+2 for slack).
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


def lut_bound(Qn, T16n, X16n):
    n = Qn.shape[1]
    Wd = np.take_along_axis(T16n.astype(np.float64), Qn.astype(np.int64), axis=1)
    mag = np.abs(X16n.astype(np.float64)) @ np.abs(Wd).T  # p x m
    return (8 * ((n + 255) // 256) + 7) * 2.0 ** -24 * mag


@pytest.mark.parametrize("nbits", list(range(1, 9)))
@pytest.mark.parametrize("m,n", [(3, 1), (5, 7), (17, 131), (64, 4096)])
def test_pack_bitwise(nbits, m, n):
    rng = np.random.default_rng(nbits * 31 + n)
    Qn = rng.integers(0, 2 ** nbits, size=(m, n), dtype=np.uint8)
    P = g.pack_codes(torch.from_numpy(Qn).to(DEV), nbits)
    assert np.array_equal(P.cpu().numpy(), oracle.pack(Qn, nbits))


def test_pack_rejects_out_of_range_codes():
    Q = torch.zeros((4, 16), dtype=torch.uint8, device=DEV)
    Q[2, 3] = 16
    with pytest.raises(ValueError):
        g.pack_codes(Q, 4)


def test_codebook_f16_bitwise():
    T = torch.from_numpy(np.random.default_rng(3).normal(size=(300, 16)).astype(np.float32) * 7.3)
    T16 = g.codebook_f16(T.to(DEV))
    assert np.array_equal(T16.cpu().numpy().view(np.uint16), T.numpy().astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("m,n,p,nbits", [
    # generic kernel (n not a multiple of 256)
    (100, 300, 3, 3), (33, 131, 8, 2), (17, 1000, 12, 8), (9, 520, 2, 5),
    # fast paths: N = 4 (direct words) and every other N (shuffled windows), n % 256 == 0
    (64, 4096, 1, 4), (40, 256, 5, 1), (64, 4096, 1, 3), (32, 512, 3, 5), (16, 768, 9, 8),
    (8, 256, 1, 2), (24, 1024, 4, 6), (10, 512, 2, 7), (300, 11008, 1, 3)])
def test_lut_gemm_parity(m, n, p, nbits):
    rng = np.random.default_rng(m * 7 + n + p)
    Qn = rng.integers(0, 2 ** nbits, size=(m, n), dtype=np.uint8)
    T16n = (rng.normal(size=(m, 2 ** nbits)) * 0.05).astype(np.float16)
    X16n = rng.normal(size=(p, n)).astype(np.float16)
    Pn = oracle.pack(Qn, nbits)
    Y = g.lut_gemm(torch.from_numpy(Pn).to(DEV), torch.from_numpy(T16n).to(DEV), torch.from_numpy(X16n).to(DEV), n)
    Yo = oracle.lut_gemm(Pn, T16n, X16n, m, n, nbits)
    err = np.abs(Y.cpu().numpy().astype(np.float64) - Yo)
    assert np.all(err <= lut_bound(Qn, T16n, X16n) + 1e-30)
    # reproducible run to run
    Y2 = g.lut_gemm(torch.from_numpy(Pn).to(DEV), torch.from_numpy(T16n).to(DEV), torch.from_numpy(X16n).to(DEV), n)
    assert torch.equal(Y, Y2)


def test_lut_gemm_identity_layer_exact():
    n = 300
    Qn = np.eye(n, dtype=np.uint8)
    T16 = torch.tensor([[0.0, 1.0]] * n, dtype=torch.float16, device=DEV)
    X = torch.from_numpy(np.random.default_rng(5).normal(size=(3, n)).astype(np.float16)).to(DEV)
    Y = g.lut_gemm(g.pack_codes(torch.from_numpy(Qn).to(DEV), 1), T16, X, n)
    assert torch.equal(Y, X.float())


def test_lut_gemm_on_quantizer_output():
    """(Q, T) from ganq_quantize_layer at c2 width, packed and served by the LUT kernel."""
    m, n, nbits = 96, 4096, 4
    W = synthetic.make_weights(m, n, seed=11).to(DEV)
    X = synthetic.make_activations(4096, n, seed=12).to(DEV)
    Q, T = g.quantize_layer(W, g.hessian(X), nbits, 2)
    P, T16 = g.pack_codes(Q, nbits), g.codebook_f16(T)
    x16 = X[:2].to(torch.float16)
    Y = g.lut_gemm(P, T16, x16, n)
    Qn, T16n, x16n = Q.cpu().numpy(), T16.cpu().numpy(), x16.cpu().numpy()
    Yo = oracle.lut_gemm(oracle.pack(Qn, nbits), T16n, x16n, m, n, nbits)
    assert np.array_equal(P.cpu().numpy(), oracle.pack(Qn, nbits))
    assert np.all(np.abs(Y.cpu().numpy() - Yo) <= lut_bound(Qn, T16n, x16n) + 1e-30)
