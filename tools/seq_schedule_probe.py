"""PA schedule sweep on the single-sequence configs (1, 2, 3, 5): ms per
sequence for fast-kernel CTAs per SM and the hybrid at low wide-step
thresholds, set through me_tuning; every variant's records are compared with
the first.  usage: seq_schedule_probe.py [config ...] [name:field=v,... ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

CONFIGS = [int(x) for x in sys.argv[1:] if ":" not in x and x.isdigit()] or [2, 3, 5]
VARIANTS = [x for x in sys.argv[1:] if not x.isdigit()]  # name:field=v,... (tuning); first one is the reference
for cid in CONFIGS:
    luma, alpha = synth.config4_batch_dev(1, 20260000, None, config_id=cid)
    F, H, W = luma.shape[1:]
    cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16 if cid <= 2 else (32 if cid == 3 else 64), block_size=8))
    res, first = {}, None
    variants = [(spec.partition(":")[0], {k: int(v) for k, v in (x.split("=") for x in spec.partition(":")[2].split(",") if x)})
                for spec in VARIANTS] if VARIANTS else \
        (("auto", {}), ("fast2", dict(pa_schedule="fast", pa_fast_ctas=2)), ("fast3", dict(pa_schedule="fast", pa_fast_ctas=3)),
         ("fast4", dict(pa_schedule="fast", pa_fast_ctas=4)), ("hyb-w5", dict(pa_schedule="hybrid", pa_wide_blocks=5 * 148)),
         ("hyb-w10", dict(pa_schedule="hybrid", pa_wide_blocks=10 * 148)), ("hyb-w20", dict(pa_schedule="hybrid", pa_wide_blocks=20 * 148)))
    for name, kw in variants:
        _lib.set_tuning(0, **kw)
        recs = torch.empty((1, F - 2, H // 8, W // 8, 16), dtype=torch.uint8, device="cuda")
        stats = torch.empty((1, F - 2, 48), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 10, 4)
        if first is None:
            first = (recs.clone(), stats.clone())
        elif not (torch.equal(first[0], recs) and torch.equal(first[1], stats)):
            res[name] = "DIFFERENT"
    _lib.set_tuning(0)
    print(f"cfg{cid}", res, flush=True)
