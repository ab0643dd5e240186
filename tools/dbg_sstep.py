"""Debug: per-column code mismatches of one GPU S-step vs the oracle (same T0)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle, synthetic
import paper_2501_12956_b200 as g

oracle.build()
for (m, n, p, nbits) in [(96, 256, 3000, 4), (96, 200, 3000, 4), (64, 384, 3000, 4), (40, 130, 2000, 3)]:
    W = synthetic.make_weights(m, n, seed=m + n)
    X = synthetic.make_activations(p, n, seed=m + n + 1)
    Hn = oracle.hessian_bf16(synthetic.bf16_bits(X))
    H = torch.from_numpy(Hn).cuda()
    L = oracle.cholesky(oracle.precondition(Hn, "none")[0])
    T0 = oracle.init_codebook(W.numpy(), nbits)
    Qg, _ = g.quantize_layer(W.cuda(), H, nbits, 1, precond="none", T0=torch.from_numpy(T0).cuda())
    Qo, _ = oracle.sstep(W.numpy().astype(np.float64), L, T0.astype(np.float64))
    mis = (Qg.cpu().numpy() != Qo)
    cols = mis.sum(0)
    first = np.nonzero(cols)[0]
    print(f"m={m} n={n}: mismatches {mis.sum()} of {m*n}; columns with mismatches: {len(first)}; "
          f"rightmost bad col {first.max() if len(first) else None}; per-128-panel from right:",
          [int(cols[max(0, n - 128 * (q + 1)):n - 128 * q].sum()) for q in range((n + 127) // 128)])
