"""Time ganq_factor (precondition + blocked fp64 Cholesky) on a synthetic H at n = 4096 / 11008.

    python tools/chol_time.py [n ...]      (CHOL_TOKENS=p overrides the 4 n calibration tokens)
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import synthetic
import paper_2501_12956_b200 as g

for n in [int(a) for a in sys.argv[1:]] or [4096]:
    X = synthetic.make_activations(int(os.environ.get("CHOL_TOKENS", 4 * n)), n, seed=2000, device="cuda")
    H = g.hessian(X)
    del X
    for _ in range(2):
        g.factor(H)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    R = 5
    for _ in range(R):
        L, _ = g.factor(H)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / R
    print(f"n={n}: factor {ms:.3f} ms  ({n ** 3 / 3 / ms / 1e9:.2f} TF/s of n^3/3)")
