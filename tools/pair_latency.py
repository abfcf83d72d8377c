"""Per-pair latency of the drop-in estimate_field path (host buffers in and
out, one pair per call), the reference's per-pair usage pattern."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import synth  # noqa: E402

for cid in (1, 2):
    luma, alpha = synth.config_sequence(cid, 5, 6)
    for algo, bs in ((me.Algo.PA, 8), (me.Algo.ES, 16), (me.Algo.FSS, 16)):
        cfg = me.SearchConfig(search_range=16, block_size=bs)
        prev = None
        for _ in range(3):
            f, st = me.estimate_field(algo, luma[2], luma[0], alpha[2], alpha[0], prev, cfg, me.PrsConfig())
        n = 50
        t = time.perf_counter()
        for i in range(n):
            f, st = me.estimate_field(algo, luma[2], luma[0], alpha[2], alpha[0], prev, cfg, me.PrsConfig())
        dt = (time.perf_counter() - t) / n
        print(f"cfg{cid} {algo.name:3s} bs{bs}: {dt * 1e6:8.1f} us per pair")
