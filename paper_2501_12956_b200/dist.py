"""Multi-GPU driver: token-sharded H with one NCCL all-reduce, row-sharded solve.

One process per GPU (torchrun).  The only data-path collective is the all-reduce of the
partial Hessians: rows of W are independent given H (Eq. 2), so
each rank then solves its contiguous block of m/G rows with no communication inside the
K loop.  Optional all-gathers assemble Q and T on every rank.

Determinism: token shards are cut at GANQ_HESSIAN_CHUNK boundaries, so every rank sums
whole fp32 chunk partials in fp64 and the fp64 all-reduce adds whole-rank sums; the
Cholesky factor is computed redundantly from the identical H on every rank.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

HESSIAN_CHUNK = 8192  # == GANQ_HESSIAN_CHUNK in include/ganq.h


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row block [r0, r1) of rank (sizes differ by at most one)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def shard_tokens(p: int, world: int, rank: int, chunk: int = HESSIAN_CHUNK) -> tuple[int, int]:
    """Token range [t0, t1) of rank, cut at chunk boundaries (whole chunks per rank)."""
    nchunks = (p + chunk - 1) // chunk
    c0, c1 = shard_rows(nchunks, world, rank)
    return min(p, c0 * chunk), min(p, c1 * chunk)


@dataclass
class DistResult:
    Q: torch.Tensor          # local rows (or all rows when gathered)
    T: torch.Tensor
    rows: tuple[int, int]    # this rank's row block
    H: torch.Tensor


def _gather_rows(local: torch.Tensor, m: int, world: int, group=None) -> torch.Tensor:
    """all_gather of uneven contiguous row blocks (pads to the largest block)."""
    sizes = [shard_rows(m, world, r) for r in range(world)]
    mx = max(r1 - r0 for r0, r1 in sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: r1 - r0] for b, (r0, r1) in zip(bufs, sizes)], dim=0)


def quantize_layer_distributed(W: torch.Tensor, X_local: torch.Tensor, n_bits: int, iters: int = 10, *,
                               group=None, gather: bool = True, hessian_fn=None, quantize_fn=None,
                               **opts) -> DistResult:
    """W: full m x n weights (every rank) or None-free; X_local: this rank's token shard.

    hessian_fn / quantize_fn default to the CUDA path (paper_2501_12956_b200.api); tests on
    CPU inject other callables to exercise the sharding and collective logic with gloo.
    """
    if hessian_fn is None or quantize_fn is None:
        from . import api
        hessian_fn = hessian_fn or api.hessian
        quantize_fn = quantize_fn or api.quantize_layer
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = W.shape[1]
    if X_local.shape[0] == 0:  # more ranks than token chunks: this rank contributes nothing
        H = torch.zeros((n, n), dtype=torch.float64, device=W.device)
    else:
        H = hessian_fn(X_local)
    if world > 1:
        dist.all_reduce(H, op=dist.ReduceOp.SUM, group=group)
    m = W.shape[0]
    r0, r1 = shard_rows(m, world, rank)
    if r1 > r0:
        Q, T = quantize_fn(W[r0:r1].contiguous(), H, n_bits, iters, **opts)
    else:  # more ranks than rows: this rank owns no rows but still joins the gathers
        Q = torch.empty((0, n), dtype=torch.uint8, device=W.device)
        T = torch.empty((0, 1 << int(n_bits)), dtype=torch.float32, device=W.device)
    if gather and world > 1:
        Q = _gather_rows(Q, m, world, group)
        T = _gather_rows(T, m, world, group)
    return DistResult(Q=Q, T=T, rows=(r0, r1), H=H)
