import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle
import paper_2501_12956_b200 as g
from test_gpu_lut import lut_bound
m, n, p, nbits = 64, 4096, 1, 4
rng = np.random.default_rng(m * 7 + n + p)
Qn = rng.integers(0, 2 ** nbits, size=(m, n), dtype=np.uint8)
T16n = (rng.normal(size=(m, 2 ** nbits)) * 0.05).astype(np.float16)
X16n = rng.normal(size=(p, n)).astype(np.float16)
Pn = oracle.pack(Qn, nbits)
Y = g.lut_gemm(torch.from_numpy(Pn).cuda(), torch.from_numpy(T16n).cuda(), torch.from_numpy(X16n).cuda(), n).cpu().numpy()
Yo = oracle.lut_gemm(Pn, T16n, X16n, m, n, nbits)
b = lut_bound(Qn, T16n, X16n)
err = np.abs(Y - Yo)
print("max err", err.max(), "max bound", b.max(), "violations", int((err > b).sum()), "of", err.size)
print("Y[:6]", Y[0, :6]); print("Yo[:6]", Yo[0, :6])
print("ratio err/bound", np.sort((err / b).ravel())[-5:])
