"""Debug: one LUT GEMV launch at c2 shape (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2501_12956_b200 as g
m = n = 4096
Q = torch.randint(0, 16, (m, n), dtype=torch.uint8, device="cuda")
T = torch.randn(m, 16, device="cuda")
P, T16 = g.pack_codes(Q, 4), g.codebook_f16(T)
x = torch.randn(1, n, dtype=torch.float16, device="cuda")
for _ in range(3):
    y = g.lut_gemm(P, T16, x, n)
torch.cuda.synchronize()
print("ok")
