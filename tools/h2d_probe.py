import torch, time
p, n = 262144, 4096
X = torch.empty((p, n), dtype=torch.bfloat16).pin_memory()
D = torch.empty((p, n), dtype=torch.bfloat16, device="cuda")
s1, s2, s3, s4 = (torch.cuda.Stream() for _ in range(4))
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps
def one():
    with torch.cuda.stream(s1): D.copy_(X, non_blocking=True)
def split(k, streams):
    def f():
        rows = p // k
        for i in range(k):
            with torch.cuda.stream(streams[i % len(streams)]):
                D[i*rows:(i+1)*rows].copy_(X[i*rows:(i+1)*rows], non_blocking=True)
    return f
gb = p * n * 2 / 1e9
for name, fn in [("1 stream", one), ("2 streams x 1", split(2, [s1, s2])), ("4 streams", split(4, [s1, s2, s3, s4])),
                 ("2 streams x 8 chunks", split(16, [s1, s2])), ("1 stream 16 chunks", split(16, [s1]))]:
    dt = t(fn)
    print(f"{name}: {gb / dt:.1f} GB/s")
