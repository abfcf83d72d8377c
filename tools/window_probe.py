"""pa_fast_kernel with the search window staged at claim time vs
per-candidate patches after the dependency wait (me_tuning.pa_fast_patches):
ms per run_sequences_dev call on config-4 batches of N sequences and on the
single-sequence configs (critical path), CUDA events, 20 calls after 3."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402


def timed(cfg, luma, alpha, reps=20):
    for _ in range(3):
        B.run_sequences_dev(cfg, luma, alpha)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        B.run_sequences_dev(cfg, luma, alpha)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


cases = [("cfg4", 4, n, 16) for n in (1, 8, 32, 64, 256)] + [("cfg1", 1, 1, 16), ("cfg2", 2, 1, 16), ("cfg3", 3, 1, 32)]
for name, cid, n, S in cases:
    F = {1: 10, 2: 30, 3: 60, 4: 30}[cid]
    luma, alpha = synth.config4_batch_dev(n, 20260000, F, config_id=cid)
    cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=S, block_size=8))
    res = {}
    for patches in (0, 1):
        _lib.set_tuning(0, pa_fast_patches=patches)
        res["patches" if patches else "window"] = timed(cfg, luma, alpha)
    _lib.set_tuning(0)
    print(name, n, res, flush=True)
    del luma, alpha
