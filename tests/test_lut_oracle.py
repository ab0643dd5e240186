"""Pins of the NEXT-1 oracle (packing, LUT mpGEMM, storage accounting) -- CPU only.

Each function is checked against something other than itself: the values Table 1 prints
(tests/golden/table1_storage.json), SPEC's worked packing examples, numpy's own bit packing
(np.packbits, little bit order) and a dense numpy matmul of the dequantized matrix.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_storage.json")))


def test_table1_percentages():
    for row in GOLD["rows"]:
        m, n = row["m"], row["n"]
        fp16 = oracle.storage_bytes(m, n, 4, "fp16")
        assert fp16 == 2 * m * n
        assert round(100 * oracle.storage_bytes(m, n, 4, "uniform") / fp16, 2) == row["uniform_pct"]
        assert round(100 * oracle.storage_bytes(m, n, 4, "lut") / fp16, 2) == row["lut_pct"]


@pytest.mark.parametrize("nbits", [1, 2, 3, 4, 8])
def test_lut_minus_uniform_is_codebook_overhead(nbits):
    m, n = 4096, 11008
    d = oracle.storage_bytes(m, n, nbits, "lut") - oracle.storage_bytes(m, n, nbits, "uniform")
    assert d == m * (2 * 2 ** nbits - 4)


def test_spec_packing_examples():
    ex = GOLD["spec_examples"]
    assert oracle.pack(np.array([ex["n4"]["codes"]], np.uint8), 4).tolist() == [ex["n4"]["bytes"]]
    assert oracle.pack(np.array([ex["n3"]["codes"]], np.uint8), 3).tolist() == [ex["n3"]["bytes"]]


@pytest.mark.parametrize("nbits", list(range(1, 9)))
@pytest.mark.parametrize("n", [1, 7, 64, 131])
def test_pack_matches_numpy_packbits_and_roundtrips(nbits, n):
    rng = np.random.default_rng(nbits * 1000 + n)
    m = 5
    Q = rng.integers(0, 2 ** nbits, size=(m, n), dtype=np.uint8)
    P = oracle.pack(Q, nbits)
    assert P.shape == (m, (n * nbits + 7) // 8)
    # independent formulation: each row's bits, code-major, LSB first, packed little-endian
    bits = ((Q[:, :, None] >> np.arange(nbits)[None, None, :]) & 1).reshape(m, n * nbits).astype(np.uint8)
    assert np.array_equal(P, np.packbits(bits, axis=1, bitorder="little"))
    assert np.array_equal(oracle.unpack(P, m, n, nbits), Q)


def test_pack_rejects_out_of_range():
    Q = np.zeros((3, 10), np.uint8)
    Q[1, 4] = 8
    with pytest.raises(ValueError, match="flat index 14"):
        oracle.pack(Q, 3)


def _dense(Q, T16):
    return np.take_along_axis(T16.astype(np.float64), Q.astype(np.int64), axis=1)


@pytest.mark.parametrize("nbits,m,n,p", [(4, 33, 100, 3), (3, 16, 257, 1), (2, 7, 64, 8), (8, 5, 40, 2)])
def test_lut_gemm_matches_dense_dequant(nbits, m, n, p):
    rng = np.random.default_rng(m * n + p)
    Q = rng.integers(0, 2 ** nbits, size=(m, n), dtype=np.uint8)
    T16 = rng.normal(size=(m, 2 ** nbits)).astype(np.float16)
    X16 = rng.normal(size=(p, n)).astype(np.float16)
    Y = oracle.lut_gemm(oracle.pack(Q, nbits), T16, X16, m, n, nbits)
    Yd = X16.astype(np.float64) @ _dense(Q, T16).T   # dequantization-based path (Fig. 1a left)
    np.testing.assert_allclose(Y, Yd, rtol=1e-12, atol=1e-12)


def test_lut_gemm_identity_and_zero_layers():
    n = 24
    Q = np.eye(n, dtype=np.uint8)                       # codebook {0, 1}: W~ = I
    T16 = np.tile(np.array([0.0, 1.0], np.float16), (n, 1))
    X16 = np.random.default_rng(1).normal(size=(4, n)).astype(np.float16)
    Y = oracle.lut_gemm(oracle.pack(Q, 1), T16, X16, n, n, 1)
    assert np.array_equal(Y, X16.astype(np.float64))
    Y0 = oracle.lut_gemm(oracle.pack(Q, 1), np.zeros_like(T16), X16, n, n, 1)
    assert not Y0.any()
