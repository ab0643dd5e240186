"""Multi-GPU driver: token-sharded H with exact integer all-reduces, row-sharded solve.

One process per GPU (torchrun).  Rows of W are independent given H (Eq. 2), so each rank
solves its contiguous block of m/G rows with no communication inside the K loop; the only
data-path exchange is the reduction of the partial Hessians:

  1. (P_r, E_r) = rank r's fp32 super-chunk partials of X X^T and the exponent bounds of its
     channels (ganq_hessian_partials, one pass over its tokens); all_reduce(E, MAX)  (n int32)
  2. Hfix_r = P_r rounded onto E's integer grid and summed (ganq_hessian_fixed: the packed
     lower-triangle tiles, int64); all_reduce(Hfix, SUM)                  (exact, any order)
  3. H = finalize(Hfix, E)                                                 (full fp64 matrix)

Token shards are whole GANQ_HESSIAN_SUPERCHUNKs, and integer sums are associative, so H -- and
hence L, Q and T -- is bitwise the same for every GPU count (reading R-12).  The Cholesky factor
is computed redundantly from that H on every rank.  Optional all-gathers assemble Q and T.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

SUPERCHUNK = 32768  # == GANQ_HESSIAN_SUPERCHUNK in include/ganq.h
HESSIAN_CHUNK = SUPERCHUNK  # token-shard granularity (kept name)


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row block [r0, r1) of rank (sizes differ by at most one)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def shard_tokens(p: int, world: int, rank: int, chunk: int = SUPERCHUNK) -> tuple[int, int]:
    """Token range [t0, t1) of rank, cut at super-chunk boundaries (whole super-chunks per rank)."""
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


def distributed_hessian(X_local: torch.Tensor, n: int, group=None, partials_fn=None, fixed_fn=None,
                        finalize_fn=None, fixed_size_fn=None) -> torch.Tensor:
    """H = X X^T over the tokens of all ranks, bitwise independent of the number of ranks.

    X_local: this rank's token shard (p_r x n bf16; p_r a multiple of SUPERCHUNK except on the last
    rank, possibly 0).  The callables default to the CUDA path (paper_2501_12956_b200.api); CPU
    tests inject emulations with the same contract to exercise the collectives over gloo."""
    if partials_fn is None:
        from . import api
        partials_fn, fixed_fn = api.hessian_partials, api.hessian_fixed
        finalize_fn, fixed_size_fn = api.hessian_finalize, api.hessian_fixed_size
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = X_local.device
    p_r = X_local.shape[0]
    if p_r > 0:
        P, E = partials_fn(X_local)
    else:  # more ranks than super-chunks: this rank contributes nothing
        P, E = None, torch.full((n,), -126, dtype=torch.int32, device=dev)
    if world > 1:
        dist.all_reduce(E, op=dist.ReduceOp.MAX, group=group)
    if p_r > 0:
        Hfix = fixed_fn(P, p_r, E)
    else:
        Hfix = torch.zeros(fixed_size_fn(n), dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(Hfix, op=dist.ReduceOp.SUM, group=group)
    return finalize_fn(Hfix, E)


def quantize_layer_distributed(W: torch.Tensor, X_local: torch.Tensor, n_bits: int, iters: int = 10, *,
                               group=None, gather: bool = True, quantize_fn=None, hessian_fns=None,
                               **opts) -> DistResult:
    """W: full m x n weights on every rank; X_local: this rank's token shard (shard_tokens).

    quantize_fn defaults to the CUDA path (paper_2501_12956_b200.api.quantize_layer); hessian_fns
    (dict of distributed_hessian's callables) default to it as well.  Tests on CPU inject other
    callables to exercise the sharding and collective logic with gloo."""
    if quantize_fn is None:
        from . import api
        quantize_fn = api.quantize_layer
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = W.shape[1]
    H = distributed_hessian(X_local, n, group=group, **(hessian_fns or {}))
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
