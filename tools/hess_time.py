"""Time the three Hessian kernels separately at c2 (CUDA events, warm)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic
import paper_2501_12956_b200 as g

dev = "cuda:0"
n, p = 4096, 262144
X = synthetic.make_activations(p, n, seed=2000, device=dev)
P, E = g.hessian_partials(X)
Hf = g.hessian_fixed(P, p, E)
H = g.hessian_finalize(Hf, E)
H2 = torch.empty_like(H)
torch.cuda.synchronize()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print("hessian_partials ms", t(lambda: g.hessian_partials(X, P=P, E=E)))
print("hessian_fixed ms", t(lambda: g.hessian_fixed(P, p, E, Hfix=Hf)))
print("hessian_finalize ms", t(lambda: g.hessian_finalize(Hf, E, H=H)))
print("hessian (all) ms", t(lambda: g.hessian(X, H=H2)))
