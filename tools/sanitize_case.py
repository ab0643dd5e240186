"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck): the whole hot path --
ganq_hessian (CTA-pair tcgen05 + exponent scan), ganq_quantize_layer (Cholesky, S-step with
cluster multicast + mbarriers + named barriers, T-step tcgen05) -- on config c1 and on a
256 x 1024 case with several panels, and a 3-bit T-update on 200 x 384."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2501_12956_b200 as g  # noqa: E402

dev = "cuda:0"
for (m, n, p, nbits, K) in [(64, 128, 256, 3, 2), (256, 1024, 40000, 4, 2), (200, 384, 3000, 3, 1)]:
    W = synthetic.make_weights(m, n, seed=1000).to(dev)
    X = synthetic.make_activations(p, n, seed=2000).to(dev)
    H = g.hessian(X)
    Q, T = g.quantize_layer(W, H, nbits, K)
    f = g.objective(W, Q, T, H)
    torch.cuda.synchronize()
    print(f"m={m} n={n} p={p} N={nbits} K={K}: objective {f:.6e}", flush=True)
print("sanitize cases done")
