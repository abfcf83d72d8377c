"""PCIe on the GPU box: H2D alone, D2H alone and both at once (two streams),
pinned buffers of the config-4 e2e sizes (0.80 GB in, 0.18 GB out)."""
import time

import torch

hin = torch.empty(802 << 20, dtype=torch.uint8).pin_memory()
hout = torch.empty(182 << 20, dtype=torch.uint8).pin_memory()
din = torch.empty_like(hin, device="cuda")
dout = torch.empty_like(hout, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                din.copy_(hin, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                hout.copy_(dout, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


run(True, True, 2)
a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D 802 MiB {a:.2f} ms ({802 * 1.048576 / a:.1f} GB/s); D2H 182 MiB {b:.2f} ms ({182 * 1.048576 / b:.1f} GB/s); both {c:.2f} ms")
