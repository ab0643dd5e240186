"""GANQ (arxiv 2501.12956) layer-wise LUT quantization solver for B200 (sm_100a).

Public API (torch CUDA tensors; thin binding of include/ganq.h):
    hessian(X)                         H = X X^T
    hessian_partials / hessian_fixed / hessian_finalize    the exact fixed-point path for token shards
    quantize_layer(W, H, n_bits, iters) -> (Q, T)            Algorithm 1
    objective(W, Q, T, H)              ||WX - W~X||_F^2      Eq. (1)
    tstep(W, Q, H, n_bits)             closed-form T-update  Eq. (6)
    factor(H)                          L = chol(H')          Eq. (9) + App. A
    dist.quantize_layer_distributed    token-sharded H + row-sharded solve over NCCL
    pack_codes / codebook_f16 / lut_gemm   NEXT-1: N-bit storage and LUT mpGEMM (Fig. 1a)
    outlier_split / sparse_gemm_add        NEXT-2: GANQ* decomposition (Algorithm 2)
    kmeans_codebook                        NEXT-4: k-means T^0 (quantize_layer(init="kmeans"))
    quantize_stacked                       NEXT-3: linears sharing H (q/k/v, gate/up) solved as one
"""
from .api import (hessian_partials, hessian_finalize, hessian_fixed, hessian_fixed_size, codebook_f16, factor, kmeans_codebook, hessian, lut_gemm, objective, objective_workspace_size, outlier_split,
                  pack_codes, quantize_layer, quantize_stacked, sparse_gemm_add, tstep, version, workspace_size)
from ._lib import GanqError, NotPositiveDefinite

__all__ = ["hessian", "hessian_partials", "hessian_fixed", "hessian_finalize", "hessian_fixed_size", "quantize_layer", "objective", "tstep", "factor", "workspace_size",
           "objective_workspace_size", "version", "pack_codes", "codebook_f16", "lut_gemm", "outlier_split",
           "sparse_gemm_add", "kmeans_codebook", "quantize_stacked", "GanqError",
           "NotPositiveDefinite"]
