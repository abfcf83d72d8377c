"""Config-4 host path: e2e time per batch, the PCIe floor, the host packing time
of one chunk's binary masks (me_b200_pack_mask, all host threads), and e2e
at several pipeline chunk counts (tuning h2d_chunks)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

n = 256
luma_d, alpha_d = synth.config4_batch_dev(n, 20260000, 30)
pin = torch.empty((2, n, 30, 288, 352), dtype=torch.uint8, pin_memory=True)
pin[0].copy_(luma_d)
pin[1].copy_(alpha_d)
hl, ha = pin[0].numpy(), pin[1].numpy()
recs = torch.empty((n, 28, 36, 44, 16), dtype=torch.uint8, pin_memory=True)
stats = torch.empty((n, 28, 48), dtype=torch.uint8, pin_memory=True)
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
# host packing of one 16-sequence chunk
chunk = ha[:16].reshape(-1)
out = np.empty(chunk.size // 8 + (1 << 20), np.uint8)
nb = C.c_size_t()
for _ in range(2):
    _lib.check(_lib.lib().me_b200_pack_mask(chunk.ctypes.data, chunk.size, out.ctypes.data, out.size, C.byref(nb)))
t = time.perf_counter()
for _ in range(5):
    _lib.check(_lib.lib().me_b200_pack_mask(chunk.ctypes.data, chunk.size, out.ctypes.data, out.size, C.byref(nb)))
print(f"pack one 16-sequence chunk ({chunk.size / 1e6:.1f} MB of mask bytes -> {nb.value / 1e6:.2f} MB): {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
for chunks in (8, 16, 32):
    _lib.set_tuning(0, h2d_chunks=chunks)
    B.run_sequences_ptr(cfg, n, 30, 352, 288, hl.ctypes.data, ha.ctypes.data, recs.data_ptr(), stats.data_ptr(), 0)
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        B.run_sequences_ptr(cfg, n, 30, 352, 288, hl.ctypes.data, ha.ctypes.data, recs.data_ptr(), stats.data_ptr(), 0)
        ts.append(time.perf_counter() - t)
    h2d, d2h = B.last_transfer_bytes(0)
    print(f"h2d_chunks {chunks}: e2e min {min(ts) * 1e3:.2f} median {np.median(ts) * 1e3:.2f} ms; H2D {h2d / 1e6:.0f} MB, D2H {d2h / 1e6:.0f} MB")
_lib.set_tuning(0)
