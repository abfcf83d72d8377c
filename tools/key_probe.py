"""PA pipeline variants on config-4 batches (me_tuning fields): ms per step,
stage times (classify, sort, search) and a check that every variant gives the
records and stats of the first.
usage: key_probe.py N[,N..] name:field=v,field=v ...   (name "default": no fields)"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
sizes = [int(x) for x in sys.argv[1].split(",")]
variants = []
for spec in sys.argv[2:] or ["default", "plain:pa_key_plain=1"]:
    name, _, kv = spec.partition(":")
    variants.append((name, {k: int(v) for k, v in (x.split("=") for x in kv.split(",") if x)}))


def stages(run):
    lib, h = _lib.lib(), _lib.ctx(0)
    _lib.check(lib.me_b200_ctx_set_profiling(h, 1))
    acc = [0.0] * 4
    for _ in range(5):
        run()
        torch.cuda.synchronize()
        st = (C.c_float * 4)()
        _lib.check(lib.me_b200_ctx_stage_ms(h, st, 4))
        acc = [a + x / 5 for a, x in zip(acc, st)]
    _lib.check(lib.me_b200_ctx_set_profiling(h, 0))
    return [round(a, 4) for a in acc[:3]]


for n in sizes:
    luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
    res, outs = {}, {}
    for name, kw in variants:
        recs = torch.empty((n, 28, 36, 44, 16), dtype=torch.uint8, device="cuda")
        stats = torch.empty((n, 28, 48), dtype=torch.uint8, device="cuda")
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
        res[name] = (round(e0.elapsed_time(e1) / 20, 4), stages(lambda: B.run_sequences_dev(cfg, luma, alpha, recs, stats)))
        outs[name] = (recs, stats)
    _lib.set_tuning(0)
    first = outs[variants[0][0]]
    same = all(torch.equal(o[i], first[i]) for o in outs.values() for i in range(2))
    print(n, res, "identical" if same else "DIFFERENT", flush=True)
    del luma, alpha, outs
