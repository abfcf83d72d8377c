import sys, torch, json
sys.path.insert(0, '.')
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import batch as B, synth, _lib
import ctypes as C
lib = me.lib(); cx = _lib.ctx(0); st = (C.c_float*4)()
for cid, S in ((5, 64), (3, 32)):
    luma, alpha = synth.config4_batch_dev(1, 20260000, 10, config_id=cid)
    for algo in ("TSS", "FSS", "DS"):
        cfg = me.BatchConfig(algo=me.Algo[algo], search=me.SearchConfig(search_range=S, block_size=16))
        res = {}
        for ctas in (4, 3, 2):
            _lib.set_tuning(0, ring_ctas=ctas)
            for _ in range(3): B.run_sequences_dev(cfg, luma, alpha)
            _lib.check(lib.me_b200_ctx_set_profiling(cx, 1))
            tot = 0
            for _ in range(10):
                B.run_sequences_dev(cfg, luma, alpha); _lib.check(lib.me_b200_ctx_stage_ms(cx, st, 4)); tot += st[2]
            _lib.check(lib.me_b200_ctx_set_profiling(cx, 0))
            res[ctas] = round(tot / 10, 4)
        print(f"cfg{cid} {algo} search ms by ring_ctas:", res, flush=True)
