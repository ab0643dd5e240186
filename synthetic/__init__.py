"""Seeded synthetic inputs for GANQ (shared by the oracle tests, the CUDA tests and bench.py).

This module holds NO arithmetic of the method -- only random draws with the
shapes and value distributions of the paper's workloads (recipe in DESIGN.md,
"Input recipe"):

* W (m x n fp32): 0.02 * N(0, 1); entries hit by a Bernoulli(0.005) mask are
  scaled x10 -- the Gaussian-plus-outlier shape of LLM weights (Fig. 1b,
  P:44-47) with the paper's 0.5 % outlier ratio.
* X (p x n bf16, token-major): x_t = (g_t + 0.5 U z_t) * s with g_t ~ N(0, I_n),
  U ~ N(0,1)^{n x 16}, z_t ~ N(0, I_16) (correlated channels) and a per-channel
  scale s_c = exp(0.5 N(0,1)) with 4 "massive" channels x30.  p = 128 x 2048
  calibration tokens for LLaMA, generated in fixed chunks.

Everything is drawn with ``torch.Generator`` seeded per tensor, on the
requested device (CPU generators for the oracle-sized cases, CUDA generators
for the full-size benchmark; the two streams differ, so each comparison uses
one stream and hands the same bytes to both sides).
"""
from __future__ import annotations

import numpy as np
import torch

# BASELINE.json configs (shapes only).  p = tokens, m x n = W.
CONFIGS = {
    "c1": dict(m=64, n=128, nbits=3, p=256, iters=10,
               desc="single synthetic linear 64x128, 3-bit, X=128x256 tokens, 10 alternating iters"),
    "c2": dict(m=4096, n=4096, nbits=4, p=128 * 2048, iters=10,
               desc="LLaMA-2-7B q_proj 4096x4096, 4-bit, 128x2048 calibration tokens, 1 B200"),
    "c3": dict(m=4096, n=11008, nbits=3, p=128 * 2048, iters=10,
               desc="LLaMA-2-7B down_proj 4096x11008, 3-bit, rows sharded over 2/4/8 B200"),
}

X_CHUNK = 32768  # generation chunk (tokens); independent of the Hessian's accumulation chunk


def make_weights(m: int, n: int, seed: int = 1000, device="cpu") -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    W = torch.randn((m, n), generator=g, device=device, dtype=torch.float32) * 0.02
    mask = torch.rand((m, n), generator=g, device=device) < 0.005
    W = torch.where(mask, W * 10.0, W)
    return W.contiguous()


def make_activations(p: int, n: int, seed: int = 2000, device="cpu", rank: int = 16,
                     n_massive: int = 4) -> torch.Tensor:
    """Token-major bf16 activations, p x n."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    U = torch.randn((n, rank), generator=g, device=device, dtype=torch.float32)
    s = torch.exp(0.5 * torch.randn((n,), generator=g, device=device, dtype=torch.float32))
    if n_massive:
        idx = torch.randperm(n, generator=g, device=device)[: min(n_massive, n)]
        s[idx] *= 30.0
    X = torch.empty((p, n), device=device, dtype=torch.bfloat16)
    for t0 in range(0, p, X_CHUNK):
        t1 = min(p, t0 + X_CHUNK)
        gt = torch.randn((t1 - t0, n), generator=g, device=device, dtype=torch.float32)
        zt = torch.randn((t1 - t0, rank), generator=g, device=device, dtype=torch.float32)
        X[t0:t1] = ((gt + 0.5 * (zt @ U.T)) * s).to(torch.bfloat16)
    return X


def make_gaussian_activations(p: int, n: int, seed: int = 3000, device="cpu") -> torch.Tensor:
    """i.i.d. N(0,1) activations (token-major bf16) -- a second, uncorrelated X shape."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((p, n), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)


def bf16_bits(X: torch.Tensor) -> np.ndarray:
    """uint16 bit patterns of a bf16 tensor (for handing the exact bytes to the oracle)."""
    assert X.dtype == torch.bfloat16
    return X.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def bf16_to_f64(X: torch.Tensor) -> np.ndarray:
    return X.detach().cpu().to(torch.float64).numpy()


def alphabet_weights(m: int, n: int, nbits: int, seed: int = 4000) -> tuple[np.ndarray, np.ndarray]:
    """Rows drawn from a per-row 2^N-value alphabet; returns (W fp32, alphabet fp32 m x 2^N)."""
    rng = np.random.default_rng(seed)
    nlev = 1 << nbits
    A = np.sort(rng.normal(0.0, 0.05, size=(m, nlev)).astype(np.float32), axis=1)
    idx = rng.integers(0, nlev, size=(m, n))
    W = np.take_along_axis(A, idx, axis=1).astype(np.float32)
    return W, A
