"""PA search time vs the dependency-poll interval (me_tuning.pa_poll_ns) at
config-4 batch sizes: ms per run_sequences_dev call (classify + sort +
search), CUDA events, 20 calls after 3 warm-up calls."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
ns_list = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "16", "64", "256"])]
for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "32", "256"])]:
    luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
    recs = torch.empty((n, 28, 36, 44, 16), dtype=torch.uint8, device="cuda")
    stats = torch.empty((n, 28, 48), dtype=torch.uint8, device="cuda")
    res = {}
    for ns in ns_list:
        _lib.set_tuning(0, pa_poll_ns=ns)
        for _ in range(3):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats)
        e1.record()
        torch.cuda.synchronize()
        res[ns] = round(e0.elapsed_time(e1) / 20, 4)
    _lib.set_tuning(0)
    print(n, res, flush=True)
    del luma, alpha, recs, stats
