import ctypes, sys, torch, subprocess
sys.path.insert(0, ".")
import synthetic
import paper_2501_12956_b200 as g
from paper_2501_12956_b200 import _lib
lib = _lib.load()
n, m = 11008, 4096
X = synthetic.make_activations(262144, n, seed=2000, device="cuda")
W = synthetic.make_weights(m, n, seed=1000, device="cuda")
def prof(fn):
    lib.ganq_profile_enable(1)
    fn(); torch.cuda.synchronize()
    ms = (ctypes.c_double * 32)(); ln = (ctypes.c_int64 * 32)()
    k = lib.ganq_profile_read(ms, ln, 32)
    lib.ganq_profile_enable(0)
    return {lib.ganq_profile_stage_name(i).decode(): round(ms[i], 2) for i in range(k) if ms[i] > 0 and lib.ganq_profile_stage_name(i).decode() in ("hessian","cholesky","sstep","tgram")}
for it in range(4):
    r = prof(lambda: g.quantize_layer(W, g.hessian(X), 3, 10))
    clk = subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
    print(it, r, clk)
H = g.hessian(X)
print("factor alone after:", prof(lambda: g.factor(H)))
