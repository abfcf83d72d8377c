#!/usr/bin/env python3
"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck):
every kernel family once, on tiny inputs (the tools slow kernels ~100x).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import synth  # noqa: E402


def run(algo, bs, S, luma, alpha, **kw):
    cfg = me.BatchConfig(algo=me.Algo[algo], search=me.SearchConfig(search_range=S, block_size=bs, halfpel=kw.get("halfpel", False)))
    r, s = me.run_sequences(cfg, luma, alpha)
    print(algo, bs, S, kw, "est blocks", int((r["type"] != 0).sum()), "cmp", int(s["block_comparisons"].sum()), flush=True)


def main():
    luma, alpha = synth.config4_batch(3, 55, 4)
    from paper_1002_1168_b200 import _lib

    for mode in ("hybrid", "fast", "warp"):
        prev = _lib.set_tuning(0, pa_schedule=mode)
        run("PA", 8, 16, luma, alpha, mode=mode)
        _lib.restore_tuning(prev, 0)
    l1, a1 = synth.config_sequence(1, 9, 4)
    run("PA", 8, 16, l1[None, :3], a1[None, :3])  # one QCIF pair: the shared-memory kernel
    run("PA", 16, 16, l1[None], a1[None], halfpel=True)
    for algo in ("ES", "TSS", "FSS", "DS"):
        run(algo, 16, 16, luma[:1], alpha[:1])
    print("sanitize_run done")


if __name__ == "__main__":
    main()
