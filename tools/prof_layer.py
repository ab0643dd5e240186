"""One c2 layer (H + quantize_layer with K = 2) on cuda:0: a short program for ncu captures.

    python tools/prof_layer.py            # exits 0 after one warm-up layer and one profiled layer
    ncu --set full -k regex:tgram_tc -s 2 -c 1 ... python tools/prof_layer.py

The hot kernels launch once per iteration (tgram_tc, sstep_tc) or once per layer (hessian_syrk),
so `-s` skips the warm-up layer's launches.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2501_12956_b200 as g  # noqa: E402


def main():
    c = synthetic.CONFIGS["c2"]
    m, n, p, nbits = c["m"], c["n"], c["p"], c["nbits"]
    dev = "cuda:0"
    W = synthetic.make_weights(m, n, seed=1000, device=dev)
    X = synthetic.make_activations(p, n, seed=2000, device=dev)
    for _ in range(2):
        H = g.hessian(X)
        Q, T = g.quantize_layer(W, H, nbits, 2)
        torch.cuda.synchronize()
    print("ok", float(T.abs().max()))


if __name__ == "__main__":
    main()
