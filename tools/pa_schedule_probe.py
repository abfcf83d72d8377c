"""PA schedule sweep over config-4 batch sizes (the per-GPU shard of the
strong-scaled runs: 256 / N sequences): ms per step for kernel schedules
and fast-kernel CTAs per SM, set through me_tuning."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
for n in [int(x) for x in (sys.argv[1:] or ["16", "32", "64", "128"])]:
    luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
    recs = torch.empty((n, 28, 36, 44, 16), dtype=torch.uint8, device="cuda")
    stats = torch.empty((n, 28, 48), dtype=torch.uint8, device="cuda")
    res = {}
    for name, kw in (("auto", {}), ("fast1", dict(pa_schedule="fast", pa_fast_ctas=1)), ("fast2", dict(pa_schedule="fast", pa_fast_ctas=2)),
                     ("fast4", dict(pa_schedule="fast", pa_fast_ctas=4)), ("hybrid", dict(pa_schedule="hybrid")),
                     ("hybrid-w20", dict(pa_schedule="hybrid", pa_wide_blocks=20 * 148)),
                     ("hybrid-w10", dict(pa_schedule="hybrid", pa_wide_blocks=10 * 148)),
                     ("duo", dict(pa_schedule="duo")), ("duo-hybrid", dict(pa_schedule="duo-hybrid")),
                     ("duo-hybrid-w10", dict(pa_schedule="duo-hybrid", pa_wide_blocks=10 * 148))):
        _lib.set_tuning(0, **kw)
        for _ in range(3):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 20, 4)
    _lib.set_tuning(0)
    print(n, res, flush=True)
    del luma, alpha, recs, stats
