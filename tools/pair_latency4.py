"""Per-pair latency split (C call vs device stages) on a QCIF noise pair."""
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import _lib
from paper_1002_1168_b200.api import _cfg, _ptr
rng = np.random.default_rng(1)
base = rng.integers(0, 256, size=(200, 240), dtype=np.uint8)
fr = [np.ascontiguousarray(base[8 + t: 8 + t + 144, 8 + 2 * t: 8 + 2 * t + 176]) for t in range(3)]
L = me.lib(); ctx = _lib.ctx()
L.me_b200_ctx_set_profiling(ctx, 1)
for algo, bs in ((me.Algo.PA, 8), (me.Algo.ES, 16)):
    cfg = _cfg(algo, me.SearchConfig(search_range=7, block_size=bs), me.PrsConfig(), 0)
    cols, rows = 176 // bs, 144 // bs
    recs = np.zeros(cols * rows, _lib.rec_dtype()); st = np.zeros(1, _lib.stats_dtype())
    args = (ctx, C.byref(cfg), 176, 144, _ptr(fr[1]), _ptr(fr[0]), None, None, None, cols, rows, _ptr(recs), _ptr(st))
    out = (C.c_float * 4)()
    for _ in range(5):
        L.me_b200_estimate_field(*args)
    t = time.perf_counter()
    for _ in range(50):
        L.me_b200_estimate_field(*args)
    dt = (time.perf_counter() - t) / 50
    L.me_b200_ctx_stage_ms(ctx, out, 4)
    print(algo.name, "call %.1f us" % (dt * 1e6), "stages us", [round(x * 1e3, 1) for x in out], "est blocks", int(st["blocks_opaque"][0]), "dpd", int(st["dpd_refinement_steps"][0]))
