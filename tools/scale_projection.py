"""Projected N-GPU layer time from measured per-rank work on ONE B200 (no multi-GPU box here).

For G = 1, 2, 4, 8 every rank runs the same work: H partials over its token
shard (p / G tokens, whole super-chunks), the fixed-point sum of its partials, the finalisation,
and ganq_quantize_layer on its m / G rows (the factorisation is replicated).  This script times
rank 0's share of each step with CUDA events on one GPU and adds the two all-reduces, estimated
from the guide's measured NVLink figure (8-rank all-reduce bus bandwidth 725 GB/s at 1 GiB):
t = bytes * 2 (G - 1) / G / 725e9 (ring-equivalent; NVLS would be faster).  The per-rank shares are
what the max over ranks takes (shards are equal sized).

    python tools/scale_projection.py [--config c3]   -> JSON lines per G and a summary
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2501_12956_b200 as g  # noqa: E402
from paper_2501_12956_b200 import _lib  # noqa: E402
from paper_2501_12956_b200.dist import shard_rows, shard_tokens  # noqa: E402

BUSBW = 725e9


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--gpus", default="1,2,4,8")
    args = ap.parse_args()
    c = synthetic.CONFIGS[args.config]
    m, n, p, nbits, K = c["m"], c["n"], c["p"], c["nbits"], c["iters"]
    dev = "cuda:0"
    W = synthetic.make_weights(m, n, seed=1000, device=dev)
    X = synthetic.make_activations(p, n, seed=2000, device=dev)
    lib = _lib.load()
    out = []
    for G in [int(x) for x in args.gpus.split(",")]:
        t0, t1 = shard_tokens(p, G, 0)
        r0, r1 = shard_rows(m, G, 0)
        Xs = X[t0:t1].contiguous()
        Ws = W[r0:r1].contiguous()
        P, E = g.hessian_partials(Xs)
        Hf = g.hessian_fixed(P, Xs.shape[0], E)
        H = g.hessian_finalize(Hf, E)
        Q = torch.empty((r1 - r0, n), dtype=torch.uint8, device=dev)
        T = torch.empty((r1 - r0, 1 << nbits), dtype=torch.float32, device=dev)
        t_part = timed(lambda: g.hessian_partials(Xs, P=P, E=E))
        t_fix = timed(lambda: g.hessian_fixed(P, Xs.shape[0], E, Hfix=Hf))
        t_fin = timed(lambda: g.hessian_finalize(Hf, E, H=H))
        lib.ganq_profile_enable(1)
        t_q = timed(lambda: g.quantize_layer(Ws, H, nbits, K, Q=Q, T=T), reps=1)
        import ctypes
        ms = (ctypes.c_double * 32)()
        ln = (ctypes.c_int64 * 32)()
        ns = int(lib.ganq_profile_read(ms, ln, 32))
        lib.ganq_profile_enable(0)
        stages = {lib.ganq_profile_stage_name(i).decode(): round(ms[i] / 2, 3) for i in range(ns) if ms[i] > 0}
        hbytes = Hf.numel() * 8
        t_ar = (hbytes * 2 * (G - 1) / G / BUSBW * 1e3) if G > 1 else 0.0
        total = t_part + t_fix + t_fin + t_q + t_ar
        rec = {"config": args.config, "G": G, "rows_per_rank": r1 - r0, "tokens_per_rank": t1 - t0,
               "hessian_partials_ms": round(t_part, 3), "hessian_fixed_ms": round(t_fix, 3),
               "hessian_finalize_ms": round(t_fin, 3), "allreduce_est_ms": round(t_ar, 3),
               "hfix_bytes": hbytes, "quantize_ms": round(t_q, 3), "quantize_stages_ms": stages,
               "rank_total_ms": round(total, 3)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del P, E, Hf, H, Q, T, Xs, Ws
        torch.cuda.empty_cache()
    base = out[0]["rank_total_ms"]
    print(json.dumps({"summary": [{"G": r["G"], "ms": r["rank_total_ms"], "speedup": round(base / r["rank_total_ms"], 2),
                                   "efficiency": round(base / r["rank_total_ms"] / r["G"], 3)} for r in out]}))


if __name__ == "__main__":
    main()
