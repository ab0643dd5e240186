import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2501_12956_b200 as g
nb = int(sys.argv[1]); m, n, p = 4, 256, 1
rng = np.random.default_rng(1)
Qn = rng.integers(0, 2 ** nb, size=(m, n), dtype=np.uint8)
T16n = (np.arange(2 ** nb)[None, :] * np.ones((m, 1))).astype(np.float16)   # t_s = s
X16n = np.zeros((p, n), np.float16)
for j in [0, 1, 7, 8, 9, 100, 255]:
    X16n[:] = 0; X16n[0, j] = 1
    Pn = oracle.pack(Qn, nb)
    Y = g.lut_gemm(torch.from_numpy(Pn).cuda(), torch.from_numpy(T16n).cuda(), torch.from_numpy(X16n).cuda(), n).cpu().numpy()
    print("j", j, "gpu codes", Y[0].astype(int).tolist(), "true", Qn[:, j].tolist())
