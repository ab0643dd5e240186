"""Isolated launches (idle gaps, no power-cap build-up) of the current Hessian at c2."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_12956_b200 as g
n, p = 4096, 262144
X = torch.full((p, n), 0.0115, dtype=torch.bfloat16, device="cuda")
H = torch.empty((n, n), dtype=torch.float64, device="cuda")
P, E = g.hessian_partials(X)
for _ in range(2):
    g.hessian(X, H=H)
torch.cuda.synchronize()
best = {}
for name, fn in (("partials", lambda: g.hessian_partials(X, P=P, E=E)), ("hessian(all)", lambda: g.hessian(X, H=H))):
    b = 1e9
    for r in range(5):
        time.sleep(0.2)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(); fn(); a1.record(); torch.cuda.synchronize()
        b = min(b, a0.elapsed_time(a1))
    print(f"current {name} best of 5: {b:.3f} ms")
