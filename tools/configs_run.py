"""BASELINE configs c4 and c5 on ONE B200, stage by stage (CUDA events, ganq_profile_*).

c4: the LLaMA-3-8B decoder layer (4-bit, K = 10, 262144 calibration tokens): q/k/v stacked
    (6144 x 4096, one H), o (4096 x 4096), gate/up stacked (28672 x 4096, one H), down
    (4096 x 14336).  Linears that read the same input share H and are solved as one problem
    (quantize_stacked, NEXT-3).
c5: the LLaMA-2-70B MLP down_proj, W 8192 x 28672, N = 3 and 4 (H over 262144 tokens).
Every layer is solved once after a warm-up of the same shape; one JSON line per layer.

    python tools/configs_run.py [c4|c5|all]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2501_12956_b200 as g  # noqa: E402
from paper_2501_12956_b200 import _lib  # noqa: E402

P_TOKENS = 128 * 2048
K = 10


def solve(name, rows, n, nbits, seed):
    dev = "cuda:0"
    lib = _lib.load()
    X = synthetic.make_activations(P_TOKENS, n, seed=seed, device=dev)
    Ws = [synthetic.make_weights(r, n, seed=seed + 1 + i, device=dev) for i, r in enumerate(rows)]
    H = torch.empty((n, n), dtype=torch.float64, device=dev)
    # warm-up (first launches, workspace, graph captures)
    g.hessian(X, H=H)
    g.quantize_stacked(Ws, H, nbits, 1)
    torch.cuda.synchronize()
    lib.ganq_profile_enable(1)
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    g.hessian(X, H=H)
    b.record()
    out = g.quantize_stacked(Ws, H, nbits, K)
    c.record()
    torch.cuda.synchronize()
    ms = (ctypes.c_double * 32)()
    ln = (ctypes.c_int64 * 32)()
    ns = int(lib.ganq_profile_read(ms, ln, 32))
    lib.ganq_profile_enable(0)
    stages = {lib.ganq_profile_stage_name(i).decode(): round(ms[i], 3) for i in range(ns) if ms[i] > 0}
    m = sum(rows)
    f = sum(g.objective(W, Q, T, H) for W, (Q, T) in zip(Ws, out))
    rec = {"layer": name, "rows": rows, "m": m, "n": n, "n_bits": nbits, "tokens": P_TOKENS, "iters": K,
           "hessian_ms": round(a.elapsed_time(b), 3), "quantize_ms": round(b.elapsed_time(c), 3),
           "total_ms": round(a.elapsed_time(c), 3), "rows_iter_per_s": round(m * K / (a.elapsed_time(c) / 1e3), 1),
           "stages_ms": stages, "objective": f}
    print(json.dumps(rec), flush=True)
    del X, Ws, H, out
    torch.cuda.empty_cache()
    return rec


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    recs = []
    if what in ("c4", "all"):
        t0 = time.time()
        recs.append(solve("c4 q/k/v (stacked)", [4096, 1024, 1024], 4096, 4, 100))
        recs.append(solve("c4 o_proj", [4096], 4096, 4, 200))
        recs.append(solve("c4 gate/up (stacked)", [14336, 14336], 4096, 4, 300))
        recs.append(solve("c4 down_proj", [4096], 14336, 4, 400))
        tot = sum(r["total_ms"] for r in recs[-4:])
        print(json.dumps({"c4_decoder_layer_ms": round(tot, 3), "wall_s": round(time.time() - t0, 1)}), flush=True)
    if what in ("c5", "all"):
        for nb in (3, 4):
            recs.append(solve(f"c5 down_proj {nb}-bit", [8192], 28672, nb, 500))


if __name__ == "__main__":
    main()
