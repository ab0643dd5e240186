"""Sequential-layer pipeline: quantize a sequence of layers held in host
memory, with the upload of layer k+1's calibration activations and weights overlapping layer
k's solve, and the download of layer k's (Q, T) overlapping layer k+1's.

Device side: two slots (X, W, H, Q, T) used alternately, a copy stream and a compute stream,
CUDA events for every hand-over; the solve is ganq_hessian + ganq_quantize_layer unchanged.
Host buffers should be pinned (page-locked) for the copies to be asynchronous.

Checkpoint / resume: quantize_layers(..., checkpoint_dir=d) writes each layer's (Q, T) to
d/layer_NNNNN.pt as soon as it is on the host (atomic rename) and, when re-run, loads the layers
already present and solves only the rest.
"""
from __future__ import annotations

import os

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

    def run(self, layers, outputs, on_done=None):
        """layers: [(W_host, X_host)], outputs: [(Q_host, T_host)] (pinned).  Each upload is
        enqueued before the previous layer's solve, so copies overlap computation.  on_done(k)
        is called on the host once layer k's outputs have arrived (layer k + 1 is queued by then)."""
        if not layers:
            return outputs
        self._upload(0, *layers[0])
        for k in range(len(layers)):
            slot = k % 2
            if k + 1 < len(layers):
                self._upload(1 - slot, *layers[k + 1])  # next layer's upload, enqueued first
            self._solve_and_download(slot, *outputs[k])
            if on_done is not None and k >= 1:
                self.down[1 - slot].synchronize()
                on_done(k - 1)
        if on_done is not None:
            self.down[(len(layers) - 1) % 2].synchronize()
            on_done(len(layers) - 1)
        return outputs

    def finish(self):
        torch.cuda.synchronize(self.dev)


def checkpoint_path(checkpoint_dir: str, k: int) -> str:
    return os.path.join(checkpoint_dir, f"layer_{k:05d}.pt")


def checkpoint_plan(n_layers: int, checkpoint_dir: str | None):
    """(done, pending) layer indices: done = those with a checkpoint file present."""
    if checkpoint_dir is None:
        return [], list(range(n_layers))
    done = [k for k in range(n_layers) if os.path.exists(checkpoint_path(checkpoint_dir, k))]
    have = set(done)
    return done, [k for k in range(n_layers) if k not in have]


def save_checkpoint(checkpoint_dir: str, k: int, Q: torch.Tensor, T: torch.Tensor, meta: dict):
    path = checkpoint_path(checkpoint_dir, k)
    tmp = path + ".tmp"
    torch.save({"Q": Q, "T": T, **meta}, tmp)
    os.replace(tmp, path)  # a layer file is either complete or absent


def load_checkpoint(checkpoint_dir: str, k: int, meta: dict):
    ck = torch.load(checkpoint_path(checkpoint_dir, k), map_location="cpu", weights_only=True)
    for key, val in meta.items():
        if ck.get(key) != val:
            raise ValueError(f"checkpoint {checkpoint_path(checkpoint_dir, k)}: {key} = {ck.get(key)!r}, "
                             f"expected {val!r}")
    return ck["Q"], ck["T"]


def quantize_layers(layers, n_bits: int, iters: int = 10, outputs=None, checkpoint_dir: str | None = None,
                    **opts):
    """[(W_host fp32 m x n, X_host bf16 p x n)] -> [(Q_host uint8, T_host fp32)], pipelined;
    with checkpoint_dir, finished layers are saved as they complete and skipped on a re-run."""
    if not layers:
        return []
    W0, X0 = layers[0]
    m, n = W0.shape
    p = X0.shape[0]
    if outputs is None:
        outputs = [(torch.empty((m, n), dtype=torch.uint8).pin_memory(),
                    torch.empty((m, 1 << n_bits), dtype=torch.float32).pin_memory()) for _ in layers]
    meta = {"m": m, "n": n, "n_bits": n_bits, "iters": iters}
    done, pending = checkpoint_plan(len(layers), checkpoint_dir)
    for k in done:
        Q, T = load_checkpoint(checkpoint_dir, k, meta)
        outputs[k][0].copy_(Q)
        outputs[k][1].copy_(T)
    if not pending:
        return outputs
    if checkpoint_dir is not None:
        os.makedirs(checkpoint_dir, exist_ok=True)

    def on_done(j):
        if checkpoint_dir is not None:
            k = pending[j]
            save_checkpoint(checkpoint_dir, k, outputs[k][0], outputs[k][1], meta)

    pipe = LayerPipeline(m, n, p, n_bits, iters, **opts)
    pipe.run([layers[k] for k in pending], [outputs[k] for k in pending], on_done=on_done)
    pipe.finish()
    return outputs
