import torch, time
n = 8 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
CH = 64 << 20
for ns in (1, 2, 3):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for j, o in enumerate(range(0, n, CH)):
            with torch.cuda.stream(ss[j % ns]):
                d[o:o + CH].copy_(h[o:o + CH], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(ns, "streams", n / dt / 1e9, "GB/s")
