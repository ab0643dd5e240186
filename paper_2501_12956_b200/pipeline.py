"""Sequential-layer pipeline: quantize a sequence of layers held in host
memory, with the upload of layer k+1's calibration activations and weights overlapping layer
k's solve, and the download of layer k's (Q, T) overlapping layer k+1's.

Device side: two slots (X, W, H, Q, T) used alternately, a copy stream and a compute stream,
CUDA events for every hand-over; the solve is ganq_hessian + ganq_quantize_layer unchanged.
Host buffers should be pinned (page-locked) for the copies to be asynchronous.
"""
from __future__ import annotations

import torch

from . import api


class LayerPipeline:
    """Pipelined GANQ over layers of one shape (m x n weights, p calibration tokens)."""

    def __init__(self, m: int, n: int, p: int, n_bits: int, iters: int = 10, device=None, **opts):
        self.dev = torch.device(device or "cuda")
        self.m, self.n, self.p, self.n_bits, self.iters, self.opts = m, n, p, n_bits, iters, opts
        self.copy = torch.cuda.Stream(self.dev)
        self.compute = torch.cuda.Stream(self.dev)
        mk = lambda shape, dt: [torch.empty(shape, dtype=dt, device=self.dev) for _ in range(2)]  # noqa: E731
        self.X = mk((p, n), torch.bfloat16)
        self.W = mk((m, n), torch.float32)
        self.H = mk((n, n), torch.float64)
        self.Q = mk((m, n), torch.uint8)
        self.T = mk((m, 1 << n_bits), torch.float32)
        self.up = [torch.cuda.Event() for _ in range(2)]     # slot uploaded
        self.done = [torch.cuda.Event() for _ in range(2)]   # slot solved
        self.down = [torch.cuda.Event() for _ in range(2)]   # slot's outputs downloaded

    def _upload(self, slot, W_host, X_host):
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.done[slot])   # the slot's previous solve has read X and W
            self.X[slot].copy_(X_host, non_blocking=True)
            self.W[slot].copy_(W_host, non_blocking=True)
            self.up[slot].record(self.copy)

    def _solve_and_download(self, slot, Q_host, T_host):
        with torch.cuda.stream(self.compute):
            self.compute.wait_event(self.up[slot])
            self.compute.wait_event(self.down[slot])  # the slot's previous outputs have left
            api.hessian(self.X[slot], H=self.H[slot], stream=self.compute)
            api.quantize_layer(self.W[slot], self.H[slot], self.n_bits, self.iters, Q=self.Q[slot], T=self.T[slot],
                               stream=self.compute, **self.opts)
            self.done[slot].record(self.compute)
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.done[slot])
            Q_host.copy_(self.Q[slot], non_blocking=True)
            T_host.copy_(self.T[slot], non_blocking=True)
            self.down[slot].record(self.copy)

    def run(self, layers, outputs):
        """layers: [(W_host, X_host)], outputs: [(Q_host, T_host)] (pinned).  Each upload is
        enqueued before the previous layer's solve, so copies overlap computation."""
        if not layers:
            return outputs
        self._upload(0, *layers[0])
        for k in range(len(layers)):
            slot = k % 2
            if k + 1 < len(layers):
                self._upload(1 - slot, *layers[k + 1])  # next layer's upload, enqueued first
            self._solve_and_download(slot, *outputs[k])
        return outputs

    def finish(self):
        torch.cuda.synchronize(self.dev)


def quantize_layers(layers, n_bits: int, iters: int = 10, outputs=None, **opts):
    """[(W_host fp32 m x n, X_host bf16 p x n)] -> [(Q_host uint8, T_host fp32)], pipelined."""
    if not layers:
        return []
    W0, X0 = layers[0]
    m, n = W0.shape
    p = X0.shape[0]
    if outputs is None:
        outputs = [(torch.empty((m, n), dtype=torch.uint8).pin_memory(),
                    torch.empty((m, 1 << n_bits), dtype=torch.float32).pin_memory()) for _ in layers]
    pipe = LayerPipeline(m, n, p, n_bits, iters, **opts)
    pipe.run(layers, outputs)
    pipe.finish()
    return outputs
