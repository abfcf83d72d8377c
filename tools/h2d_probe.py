"""H2D / D2H bandwidth of pinned copies (the e2e bound)."""
import time

import torch

n = 876 * 2**20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for chunks in (1, 16, 32):
    t = time.perf_counter()
    for _ in range(5):
        step = n // chunks
        for i in range(chunks):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"H2D {chunks} chunks: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms for {n / 2**20:.0f} MiB)")
t = time.perf_counter()
for _ in range(5):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"D2H: {n / dt / 1e9:.1f} GB/s")
