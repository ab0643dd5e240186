"""The N > 1 path with the CUDA kernels and NCCL (paper_2501_12956_b200/dist.py): world size 2 on
two GPUs of one node, one process per GPU.  Token shards are whole super-chunks, the partial
Hessians are reduced exactly (MAX of the grid exponents, int64 SUM of the fixed-point tiles), so
H, and with it every rank's rows of (Q, T), must be bitwise those of one GPU (reading R-12).

Skipped when fewer than two GPUs are visible (the round-end GPU tier has one); the same host
logic runs over gloo on CPU in tests/test_dist_cpu.py, and the G-invariance of H on one GPU in
tests/test_gpu_parity.py::test_hessian_gpu_count_invariance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic

pytestmark = pytest.mark.gpu

M, N_, P_, NBITS, K = 96, 256, 3 * 32768 + 1000, 3, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from paper_2501_12956_b200.dist import quantize_layer_distributed, shard_tokens
        W = synthetic.make_weights(M, N_, seed=21).to(dev)
        X = synthetic.make_activations(P_, N_, seed=22).to(dev)
        t0, t1 = shard_tokens(P_, world, rank)
        res = quantize_layer_distributed(W, X[t0:t1].contiguous(), NBITS, K)
        torch.cuda.synchronize()
        out[rank] = (res.H.cpu().numpy(), res.Q.cpu().numpy(), res.T.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_world2_nccl_bitwise_equals_one_gpu():
    import paper_2501_12956_b200 as g
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn", join=True)
    W = synthetic.make_weights(M, N_, seed=21).cuda()
    X = synthetic.make_activations(P_, N_, seed=22).cuda()
    H = g.hessian(X)
    Q, T = g.quantize_layer(W, H, NBITS, K)
    for r in range(world):
        Hr, Qr, Tr = out[r]
        assert np.array_equal(Hr, H.cpu().numpy())
        assert np.array_equal(Qr, Q.cpu().numpy()) and np.array_equal(Tr, T.cpu().numpy())
