"""Multi-process host logic of the multi-GPU driver (paper_2501_12956_b200/dist.py) on CPU.

World size 2 over gloo (127.0.0.1).  The per-rank compute is injected with the fp64 oracle,
so these tests exercise exactly the sharding, the all-reduce of the partial Hessians and the
gather of row blocks -- the parts of the N > 1 path that do not need a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from paper_2501_12956_b200.dist import HESSIAN_CHUNK, quantize_layer_distributed, shard_rows, shard_tokens


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
    for p in (100, HESSIAN_CHUNK, 3 * HESSIAN_CHUNK + 5, 262144):
        for world in (1, 2, 4, 8):
            rng = [shard_tokens(p, world, r) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == p
            for (a, b), (c, d) in zip(rng, rng[1:]):
                assert b == c
            for a, b in rng:
                assert a == b or a % HESSIAN_CHUNK == 0  # whole chunks: exact fp64 sums (R-12)


def _oracle_hessian(Xloc):
    import oracle
    if Xloc.shape[0] == 0:
        return torch.zeros((Xloc.shape[1], Xloc.shape[1]), dtype=torch.float64)
    return torch.from_numpy(oracle.hessian_bf16(synthetic.bf16_bits(Xloc)))


def _oracle_quantize(Wloc, H, nbits, iters, **kw):
    import oracle
    Q, T = oracle.quantize(Wloc.numpy().astype(np.float64), H.numpy(), nbits, iters)
    return torch.from_numpy(Q), torch.from_numpy(T)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, p, nbits, K = 23, 40, 3 * HESSIAN_CHUNK // 64, 3, 3
        W = synthetic.make_weights(m, n, seed=5)
        X = synthetic.make_activations(p, n, seed=6)
        t0, t1 = shard_tokens(p, world, rank, chunk=HESSIAN_CHUNK // 64)
        res = quantize_layer_distributed(W, X[t0:t1].contiguous(), nbits, K,
                                         hessian_fn=_oracle_hessian, quantize_fn=_oracle_quantize)
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
    m, n, p, nbits, K = 23, 40, 3 * HESSIAN_CHUNK // 64, 3, 3
    W = synthetic.make_weights(m, n, seed=5)
    X = synthetic.make_activations(p, n, seed=6)
    Hfull = oracle.hessian_bf16(synthetic.bf16_bits(X))
    Q0, T0, H0, rows0 = out[0]
    Q1, T1, H1, rows1 = out[1]
    assert np.array_equal(H0, H1)                      # every rank holds the same reduced H
    np.testing.assert_allclose(H0, Hfull, rtol=1e-12)  # = X X^T of all tokens
    assert rows0 == (0, 12) and rows1 == (12, 23)
    assert np.array_equal(Q0, Q1) and np.array_equal(T0, T1)  # gathered on both ranks
    Qs, Ts = oracle.quantize(W.numpy().astype(np.float64), H0, nbits, K)
    assert np.array_equal(Q0, Qs)                      # rows are independent (Eq. 2)
    np.testing.assert_array_equal(T0, Ts)
