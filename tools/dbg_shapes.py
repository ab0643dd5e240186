import torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2501_12956_b200 as g
for n in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(1)
    W = torch.from_numpy(rng.normal(size=(5, n)).astype(np.float32)).cuda()
    A = rng.normal(size=(n, 3 * n + 3)); H = torch.from_numpy(A @ A.T + np.eye(n)).cuda()
    try:
        Q, T = g.quantize_layer(W, H, 2, 2)
        torch.cuda.synchronize()
        print(n, "ok", Q.cpu().numpy().ravel()[:8])
    except Exception as e:
        print(n, "ERR", e); break
