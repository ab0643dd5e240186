"""NEXT-4: preconditioning sweep in the structure of Table 7 on the synthetic c2
layer: the objective ||WX - W~X||_F^2 after K = 10 iterations (instead of WikiText-2 perplexity,
which needs a model and data) for H + lambda p I with lambda in {0.5, 1, 10, 40, 100} (Table 7's
values for the normalised Hessian XX^T / p, reading R-23), the adaptive method of Eqs. 23-24,
no preconditioning, and "auto" (none unless the factor fails); plus both empty-level rules and
the k-means initial codebook (R-24).

    python tools/precond_sweep.py [--rows 4096] > profiles/r01_precond_sweep.md
"""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import synthetic
import paper_2501_12956_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--config", default="c2")
args = ap.parse_args()
c = synthetic.CONFIGS[args.config]
m, n, p, nbits, K = min(args.rows, c["m"]), c["n"], c["p"], c["nbits"], c["iters"]
W = synthetic.make_weights(c["m"], n, seed=1000, device="cuda")[:m].contiguous()
X = synthetic.make_activations(p, n, seed=2000, device="cuda")
H = g.hessian(X)
del X
rows = []


def run(name, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Q, T, trace = g.quantize_layer(W, H, nbits, K, trace=True, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rows.append({"policy": name, "objective": trace[-1], "trace": trace, "s": dt})


for lam in (0.5, 1.0, 10.0, 40.0, 100.0):
    run(f"fixed lambda = {lam:g} (x p)", precond="fixed_lambda", lam=lam * p)
run("adaptive (Eqs. 23-24)", precond="adaptive")
run("none", precond="none")
run("auto (none unless not PD)", precond="auto")
run("adaptive, keep-previous empty levels", precond="adaptive", empty_level_rule=1)
run("adaptive, k-means T0 (25 Lloyd iterations, R-24)", precond="adaptive", init="kmeans")
run("none, k-means T0 (25 Lloyd iterations, R-24)", precond="none", init="kmeans")
run("fixed lambda = 100 (x p), k-means T0", precond="fixed_lambda", lam=100.0 * p, init="kmeans")
best = min(r["objective"] for r in rows)
print(f"# Preconditioning sweep, {args.config}: W {m} x {n}, {nbits}-bit, p = {p}, K = {K} (synthetic, seeds 1000/2000)\n")
print("Structure of Table 7 (P:470-491); objective ||WX - W~X||_F^2 after K iterations (lower is better).\n")
print("| policy | objective | vs best | wall s |")
print("|---|---|---|---|")
for r in rows:
    print(f"| {r['policy']} | {r['objective']:.6e} | {r['objective'] / best:.4f} | {r['s']:.3f} |")
print("\n```json")
print(json.dumps([{k: v for k, v in r.items()} for r in rows]))
print("```")
