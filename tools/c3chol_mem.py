import sys, torch, subprocess
sys.path.insert(0, ".")
import synthetic
import paper_2501_12956_b200 as g
n = 11008
X = synthetic.make_activations(262144, n, seed=2000, device="cuda")
H = g.hessian(X)
def t(label):
    g.factor(H); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): g.factor(H)
    b.record(); torch.cuda.synchronize()
    clk = subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
    print(label, round(a.elapsed_time(b) / 3, 2), "ms", clk, flush=True)
t("X alive (5.8 GB)")
del X; torch.cuda.empty_cache()
t("X freed")
big = torch.empty(12 * 2**30, dtype=torch.uint8, device="cuda")
t("12 GB dummy alive")
del big; torch.cuda.empty_cache()
t("dummy freed")
