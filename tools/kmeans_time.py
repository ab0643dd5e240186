"""Time ganq_kmeans_codebook at the c2 shape (CUDA events, after warm-up)."""
import torch
import synthetic
import paper_2501_12956_b200 as g

W = synthetic.make_weights(4096, 4096, seed=1001, device="cuda")
for it in (1, 25):
    for _ in range(3):
        g.kmeans_codebook(W, 4, it)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        g.kmeans_codebook(W, 4, it)
    b.record()
    torch.cuda.synchronize()
    print(f"kmeans iters={it}: {a.elapsed_time(b) / 10:.3f} ms")
