import torch, time
n = 73289328
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(k):
    ss = [torch.cuda.Stream() for _ in range(k)]
    cs = n // k
    for _ in range(3):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    print(k, "streams", f"{n/dt/1e9:.1f} GB/s", f"{dt*1e3:.3f} ms")
for k in (1, 2, 4, 8):
    run(k)
