"""NEXT-3: q/k/v of a LLaMA-3-8B decoder layer (q 4096 x 4096, k and v 1024 x 4096, N = 4, shared
input X of 262 144 tokens) quantized as three separate layers vs one stacked 6144-row problem.

    python tools/stacked_qkv.py > profiles/r01_stacked_qkv.md
"""
import sys

import torch

sys.path.insert(0, ".")
import synthetic
import paper_2501_12956_b200 as g

n, p, nbits, K = 4096, 262144, 4, 10
X = synthetic.make_activations(p, n, seed=2000, device="cuda")
Ws = [synthetic.make_weights(m, n, seed=1000 + i, device="cuda") for i, m in enumerate((4096, 1024, 1024))]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def separate():
    for W in Ws:
        g.quantize_layer(W, g.hessian(X), nbits, K)


def stacked():
    g.quantize_stacked(Ws, g.hessian(X), nbits, K)


ts, tk = timed(separate), timed(stacked)
print("# Stacked q/k/v (SURVEY NEXT-3), LLaMA-3-8B shapes, one B200\n")
print(f"q 4096 x 4096, k 1024 x 4096, v 1024 x 4096; {nbits}-bit, K = {K}, H from {p} tokens (synthetic).\n")
print("| variant | ms | per-block result |")
print("|---|---|---|")
print(f"| three layers (3 x H, 3 x factor, 3 x solve) | {ts:.2f} | reference |")
print(f"| stacked 6144 rows (1 x H, 1 x factor, 1 x solve) | {tk:.2f} | bit-identical (tests/test_gpu_pipeline.py) |")
print(f"\nspeed-up {ts / tk:.2f}x")
