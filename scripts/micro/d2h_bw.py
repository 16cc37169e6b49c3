import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.int32, device="cuda")
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = n // parts
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(parts, "streams", 4*n/dt/1e9, "GB/s")
# H2D for reference
torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); print("h2d", 4*n/(time.perf_counter()-t)/1e9)
