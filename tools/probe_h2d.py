"""Pinned host -> device copy bandwidth with 1/2/4 concurrent streams (the e2e bound)."""
import torch, time
n = 1 << 32
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        chunk = n // ns
        for i in range(ns):
            with torch.cuda.stream(s[i]):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(ns, "streams:", round(n / (t1 - t0) / 1e9, 2), "GB/s")
# many medium copies on 2 streams alternating
for ns in (1, 2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    step = 64 << 20
    for j, off in enumerate(range(0, n, step)):
        with torch.cuda.stream(s[j % ns]):
            d[off:off+step].copy_(h[off:off+step], non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("64MB pieces on", ns, "streams:", round(n / (t1 - t0) / 1e9, 2), "GB/s")
