"""NEXT-2 (GANQ* outlier split, Algorithm 2) on the GPU vs the oracle, through the C ABI.

  split: bit-exact -- cutoffs are order statistics (selection, integer work), W_dense = W - W o M
         exactly, CSR offsets / columns / values equal the oracle's;
  sparse_gemm_add: |dy| <= (ceil(nnz_i / 32) + 7) 2^-24 sum_k |v_k x_{col_k}| (each lane adds its
         strided entries in fp32 with fused multiply-adds, then a 5-level butterfly, then the add
         into Y) plus the rounding of that final add.
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


def cases():
    rng = np.random.default_rng(7)
    out = [("synthetic", synthetic.make_weights(64, 4096, seed=21).numpy(), 0.005),
           ("t3", rng.standard_t(3, size=(33, 1000)).astype(np.float32), 0.02),
           ("ties", rng.integers(-3, 4, size=(17, 300)).astype(np.float32), 0.1),
           ("zeros", np.where(rng.random((9, 128)) < 0.5, 0.0, -0.0).astype(np.float32), 0.05),
           ("tiny", rng.normal(size=(5, 2)).astype(np.float32), 0.5),
           ("c3row", synthetic.make_weights(8, 11008, seed=22).numpy(), 0.005)]
    return out


@pytest.mark.parametrize("name,W,r", cases(), ids=[c[0] for c in cases()])
def test_outlier_split_bitwise(name, W, r):
    M, Wd_o, clo_o, chi_o = oracle.outlier_split(W, r)
    off_o, col_o, val_o = oracle.csr_of(W, M)
    Wd, (off, col, val), (clo, chi) = g.outlier_split(torch.from_numpy(W).to(DEV), r)
    assert np.array_equal(Wd.cpu().numpy().view(np.uint32), Wd_o.view(np.uint32))
    assert np.array_equal(clo.cpu().numpy(), clo_o) and np.array_equal(chi.cpu().numpy(), chi_o)
    assert np.array_equal(off.cpu().numpy(), off_o)
    assert np.array_equal(col.cpu().numpy(), col_o)
    assert np.array_equal(val.cpu().numpy().view(np.uint32), val_o.view(np.uint32))


def test_outlier_split_rejects_bad_ratio():
    W = torch.zeros((2, 8), device=DEV)
    for r in (0.0, 1.0, -0.1):
        with pytest.raises(g.GanqError):
            g.outlier_split(W, r)


@pytest.mark.parametrize("p", [1, 5])
def test_sparse_gemm_add(p):
    rng = np.random.default_rng(p)
    W = rng.standard_t(3, size=(50, 700)).astype(np.float32)
    _, csr, _ = g.outlier_split(torch.from_numpy(W).to(DEV), 0.05)
    off, col, val = csr
    X16 = rng.normal(size=(p, 700)).astype(np.float16)
    Y0 = rng.normal(size=(p, 50)).astype(np.float32)
    Y = g.sparse_gemm_add(csr, torch.from_numpy(X16).to(DEV), torch.from_numpy(Y0.copy()).to(DEV)).cpu().numpy()
    offn, coln, valn = off.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
    Ys = oracle.sparse_matmul(offn, coln, valn, 50, 700, X16.astype(np.float64))
    cnt = np.diff(offn)
    mag = np.zeros((p, 50))
    for i in range(50):
        ks = slice(offn[i], offn[i + 1])
        mag[:, i] = np.abs(X16[:, coln[ks]].astype(np.float64)) @ np.abs(valn[ks].astype(np.float64))
    bound = (np.ceil(cnt / 32) + 7) * 2.0 ** -24 * mag + 2.0 ** -24 * np.abs(Y0 + Ys)
    assert np.all(np.abs(Y - (Y0 + Ys)) <= bound + 1e-30)


def test_ganq_star_improves_on_planted_outliers():
    """GANQ* (§3.3): quantizing W_dense leaves a smaller objective than quantizing W,
    on weights with planted x10 outliers (P:242's 0.5 % ratio)."""
    m, n, nbits = 64, 512, 3
    W = synthetic.make_weights(m, n, seed=31).to(DEV)
    X = synthetic.make_activations(4096, n, seed=32).to(DEV)
    H = g.hessian(X)
    Q, T = g.quantize_layer(W, H, nbits, 5, precond="none")
    f_plain = g.objective(W, Q, T, H)
    Wd, csr, _ = g.outlier_split(W, 0.005)
    Qd, Td = g.quantize_layer(Wd, H, nbits, 5, precond="none")
    f_star = g.objective(Wd, Qd, Td, H)  # W - (W~_dense + W_sparse) = W_dense - W~_dense
    assert f_star < f_plain


def test_ganq_star_deployed_layer_matches_oracle():
    """The deployed GANQ* layer end to end: split (Algorithm 2) -> quantize W_dense -> pack ->
    fp16 codebook -> Y = LUT mpGEMM + sparse outliers, against the oracle's fp64 product of the
    same stored operands (unpacked codes, fp16 codebook, CSR of the oracle's own split).  Bound:
    the sum of the two kernels' derived bounds (tests/test_gpu_lut.py, this file's header)."""
    m, n, p, nbits = 48, 512, 3, 4
    W = synthetic.make_weights(m, n, seed=41)
    Xc = synthetic.make_activations(2048, n, seed=42).to(DEV)
    H = g.hessian(Xc)
    Wd, csr, _ = g.outlier_split(W.to(DEV), 0.005)
    Q, T = g.quantize_layer(Wd, H, nbits, 3, precond="none")
    Pk = g.pack_codes(Q, nbits)
    T16 = g.codebook_f16(T)
    X16 = (torch.randn((p, n), generator=torch.Generator().manual_seed(43)) * 0.5).to(torch.float16)
    Y = g.lut_gemm(Pk, T16, X16.to(DEV), n)
    Y = g.sparse_gemm_add(csr, X16.to(DEV), Y)
    torch.cuda.synchronize()
    # oracle side: the stored operands, the oracle's own split of W (bitwise equal, P-split)
    M, Wd_o, _, _ = oracle.outlier_split(W.numpy(), 0.005)
    assert np.array_equal(Wd_o, Wd.cpu().numpy())
    Qo = oracle.unpack(Pk.cpu().numpy(), m, n, nbits)
    assert np.array_equal(Qo, Q.cpu().numpy())
    T16o = T16.cpu().numpy().astype(np.float64)
    Wt = np.take_along_axis(T16o, Qo.astype(np.int64), axis=1)  # W~_dense (stored fp16 levels)
    Ws = np.where(M, W.numpy().astype(np.float64), 0.0)            # W_sparse
    x = X16.numpy().astype(np.float64)
    Yo = x @ (Wt + Ws).T
    absb = np.abs(x) @ (np.abs(Wt) + np.abs(Ws)).T
    bound = ((8 * -(-n // 256) + 7) + (-(-n // 32) + 8)) * 2.0 ** -24 * absb + 1e-30
    assert np.all(np.abs(Y.cpu().numpy().astype(np.float64) - Yo) <= bound)
