"""Aggregate throughput of config-4 batches run by 1 vs 2 host threads
(separate contexts and streams): do two pipelines overlap (one's classify
stream beside the other's latency-bound search) or serialise?"""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
outs = [(torch.empty((n, 28, 36, 44, 16), dtype=torch.uint8, device="cuda"), torch.empty((n, 28, 48), dtype=torch.uint8, device="cuda")) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
ITER = 40


def work(k, iters, tune):
    if tune:
        _lib.set_tuning(0, **tune)
    with torch.cuda.stream(streams[k]):
        for _ in range(iters):
            B.run_sequences_dev(cfg, luma, alpha, *outs[k], stream=streams[k].cuda_stream)
    streams[k].synchronize()


for tune in ({}, dict(pa_quad_ctas=2), dict(pa_quad_ctas=2, pa_fast_ctas=2)):
    for _ in range(3):
        work(0, 2, tune)
    torch.cuda.synchronize()
    t = time.perf_counter()
    work(0, ITER, tune)
    t1 = (time.perf_counter() - t) / ITER
    th = [threading.Thread(target=work, args=(k, ITER // 2, tune)) for k in range(2)]
    t = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    t2 = (time.perf_counter() - t) / ITER
    same = torch.equal(outs[0][0], outs[1][0])
    print(f"n={n} tune={tune}: 1 thread {t1 * 1e3:.3f} ms/batch, 2 threads {t2 * 1e3:.3f} ms/batch, identical {same}", flush=True)
