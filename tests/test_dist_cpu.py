"""Multi-process host logic of the multi-GPU driver (paper_2501_12956_b200/dist.py) on CPU.

World size 2 over gloo (127.0.0.1).  The per-rank compute is injected: the S/T solve with the fp64
oracle, the Hessian with a numpy emulation of ganq_hessian_fixed's contract (every super-chunk's
X X^T rounded onto the integer grid 2^(E_i + E_j - 31), int64 sums; reading R-12) built on the
oracle's fp64 H.  These tests exercise exactly the sharding, the MAX all-reduce of the channel
exponents, the exact int64 SUM all-reduce of the partial Hessians and the gather of row blocks --
the parts of the N > 1 path that do not need a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from paper_2501_12956_b200.dist import SUPERCHUNK, quantize_layer_distributed, shard_rows, shard_tokens


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_rows_cover_and_balance():
    for m in (1, 7, 64, 4096, 4097):
        for world in (1, 2, 3, 8):
            blocks = [shard_rows(m, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_shard_tokens_chunk_aligned():
    for p in (100, SUPERCHUNK, 3 * SUPERCHUNK + 5, 262144):
        for world in (1, 2, 4, 8):
            rng = [shard_tokens(p, world, r) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == p
            for (a, b), (c, d) in zip(rng, rng[1:]):
                assert b == c
            for a, b in rng:
                assert a == b or a % SUPERCHUNK == 0  # whole super-chunks: exact integer sums (R-12)


SC = SUPERCHUNK // 64  # emulated super-chunk (small test sizes)


def _emu_partials(Xloc):
    """(the oracle's fp64 X X^T of every super-chunk, E from their diagonals: E_c = ceil(e/2) + 1
    for max_sc P_sc[c][c] = m 2^e, m in [0.5, 1) -- the rule of ganq_hessian_partials)"""
    import oracle
    P = [oracle.hessian_bf16(synthetic.bf16_bits(Xloc[t0:t0 + SC].contiguous())) for t0 in range(0, Xloc.shape[0], SC)]
    D = np.max(np.stack([np.diag(h) for h in P]), axis=0)
    _, e = np.frexp(D)
    E = np.where(D > 0, ((e + 1) >> 1) + 1, -126).astype(np.int32)
    return P, torch.from_numpy(E)


def _emu_fixed(P, p, E):
    e = E.numpy().astype(np.int64)
    acc = np.zeros(P[0].shape, np.int64)
    for Hs in P:
        acc += np.rint(np.ldexp(Hs, 46 - e[:, None] - e[None, :])).astype(np.int64)
    return torch.from_numpy(acc.reshape(-1))


def _emu_finalize(Hfix, E):
    n = E.shape[0]
    e = E.numpy().astype(np.int64)
    return torch.from_numpy(np.ldexp(Hfix.numpy().reshape(n, n).astype(np.float64), e[:, None] + e[None, :] - 46))


EMU = dict(partials_fn=_emu_partials, fixed_fn=_emu_fixed, finalize_fn=_emu_finalize, fixed_size_fn=lambda n: n * n)


def _oracle_quantize(Wloc, H, nbits, iters, **kw):
    import oracle
    Q, T = oracle.quantize(Wloc.numpy().astype(np.float64), H.numpy(), nbits, iters)
    return torch.from_numpy(Q), torch.from_numpy(T)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, p, nbits, K = 23, 40, 3 * SC, 3, 3
        W = synthetic.make_weights(m, n, seed=5)
        X = synthetic.make_activations(p, n, seed=6)
        t0, t1 = shard_tokens(p, world, rank, chunk=SC)
        res = quantize_layer_distributed(W, X[t0:t1].contiguous(), nbits, K, hessian_fns=EMU,
                                         quantize_fn=_oracle_quantize)
        out[rank] = (res.Q.numpy(), res.T.numpy(), res.H.numpy(), res.rows)
    finally:
        dist.destroy_process_group()


def test_world2_gloo_matches_single_process():
    import oracle
    oracle.build()
    world = 2
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, start_method="spawn", join=True)
    m, n, p, nbits, K = 23, 40, 3 * SC, 3, 3
    W = synthetic.make_weights(m, n, seed=5)
    X = synthetic.make_activations(p, n, seed=6)
    Hfull = oracle.hessian_bf16(synthetic.bf16_bits(X))
    Q0, T0, H0, rows0 = out[0]
    Q1, T1, H1, rows1 = out[1]
    assert np.array_equal(H0, H1)                      # every rank holds the same reduced H
    P, E = _emu_partials(X)
    H1p = _emu_finalize(_emu_fixed(P, p, E), E).numpy()
    assert np.array_equal(H0, H1p)                     # bitwise the single-process fixed-point H
    e = E.numpy().astype(np.int64)
    grid = np.ldexp(1.0, e[:, None] + e[None, :] - 46)
    assert np.all(np.abs(H0 - Hfull) <= 3 * 0.5 * grid + 1e-15 * np.abs(Hfull))  # X X^T, one rounding per super-chunk
    assert rows0 == (0, 12) and rows1 == (12, 23)
    assert np.array_equal(Q0, Q1) and np.array_equal(T0, T1)  # gathered on both ranks
    Qs, Ts = oracle.quantize(W.numpy().astype(np.float64), H0, nbits, K)
    assert np.array_equal(Q0, Qs)                      # rows are independent (Eq. 2)
    np.testing.assert_array_equal(T0, Ts)


def _oracle_quantize_f32(Wloc, H, nbits, iters, **kw):
    Q, T = _oracle_quantize(Wloc, H, nbits, iters, **kw)
    return Q, T.float()  # the product's codebook dtype (fp32), as the empty shard's


def _worker_fewer_rows(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, p, nbits, K = 1, 24, 2 * SC, 2, 2
        W = synthetic.make_weights(m, n, seed=7)
        X = synthetic.make_activations(p, n, seed=8)
        t0, t1 = shard_tokens(p, world, rank, chunk=SC)
        res = quantize_layer_distributed(W, X[t0:t1].contiguous(), nbits, K, hessian_fns=EMU,
                                         quantize_fn=_oracle_quantize_f32)
        out[rank] = (res.Q.numpy(), res.T.numpy(), res.rows)
    finally:
        dist.destroy_process_group()


def test_world2_gloo_more_ranks_than_rows():
    """m = 1 < world = 2: rank 1 owns no rows, skips the solve and still joins the collectives
    (no hang); both ranks end with the one row's (Q, T)."""
    import oracle
    oracle.build()
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker_fewer_rows, args=(world, _free_port(), out), nprocs=world, start_method="spawn",
                       join=True)
    Q0, T0, rows0 = out[0]
    Q1, T1, rows1 = out[1]
    assert rows0 == (0, 1) and rows1 == (1, 1)
    assert Q0.shape == (1, 24) and np.array_equal(Q0, Q1) and np.array_equal(T0, T1)
