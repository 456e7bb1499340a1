"""Pinned host-to-device copy bandwidth with 1, 2 and 4 concurrent streams (e2e is bound by it)."""
import torch, time
n = 16 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(200):
        c = n // k
        for j in range(k):
            with torch.cuda.stream(ss[j]):
                d[j*c:(j+1)*c].copy_(h[j*c:(j+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(k, "streams:", round(200 * n / dt / 1e9, 1), "GB/s")
