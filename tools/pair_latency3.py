import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import synth, _lib
from paper_1002_1168_b200.api import _cfg, _ptr
luma, alpha = synth.config_sequence(1, 5, 6)
L = me.lib(); ctx = _lib.ctx()
stream = torch.cuda.ExternalStream(L.me_b200_ctx_stream(ctx)) if hasattr(torch.cuda, "ExternalStream") else None
for algo, bs in ((me.Algo.PA, 8), (me.Algo.ES, 16)):
    cfg = _cfg(algo, me.SearchConfig(search_range=16, block_size=bs), me.PrsConfig(), 0)
    cols, rows = 176 // bs, 144 // bs
    recs = np.zeros(cols * rows, _lib.rec_dtype()); st = np.zeros(1, _lib.stats_dtype())
    args = (ctx, C.byref(cfg), 176, 144, _ptr(luma[2]), _ptr(luma[0]), _ptr(alpha[2]), _ptr(alpha[0]), None, cols, rows, _ptr(recs), _ptr(st))
    for _ in range(5): L.me_b200_estimate_field(*args)
    n = 200; t = time.perf_counter()
    for _ in range(n): L.me_b200_estimate_field(*args)
    print(algo.name, "C call %.1f us" % ((time.perf_counter() - t) / n * 1e6))
