"""Per-block phase trace of the one-CTA shared-memory PA kernel (the per-pair
estimate_field path): SM clocks {wait start, ready, BRS done, walk done,
published} per block, then the per-level chain: detect (ready - last
dependency published), BRS, walk, publish.  usage: smem_trace.py [config] [pair]"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1002_1168_b200 import _lib, api, synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
f = int(sys.argv[2]) if len(sys.argv) > 2 else 4
luma, _ = synth.config_sequence(cid, 7, f + 1)
cfg, prs = api.SearchConfig(search_range=16, block_size=8), api.PrsConfig()
prev, _ = api.estimate_field(api.Algo.PA, luma[f - 1], luma[f - 3], None, None, None, cfg, prs)
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "smem_trace.bin")
for use_prev in (False, True):
    _lib.set_tuning(0, pa_trace_path=path)
    api.estimate_field(api.Algo.PA, luma[f], luma[f - 2], None, None, prev if use_prev else None, cfg, prs)
    _lib.set_tuning(0)
    H, W = luma.shape[1:]
    cols, rows = W // 8, H // 8
    tr = np.fromfile(path, np.int64).reshape(rows, cols, 5).astype(np.float64)
    t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
    tr = (tr - t0) / 1965.0  # us at 1965 MHz
    done = tr[:, :, 4]
    dep = np.full((rows, cols), -1e9)
    for v in range(rows):
        for h in range(cols):
            d = [done[v, h - 1] if h > 0 else -1e9, done[v - 1, h] if v > 0 else -1e9,
                 done[v - 1, h + 1] if v > 0 and h + 1 < cols else -1e9]
            dep[v, h] = max(d)
    has = dep > -1e8
    det = tr[:, :, 1][has] - dep[has]
    print(f"cfg{cid} pair prev={use_prev}: span {done.max():.1f} us, levels {cols - 1 + 2 * (rows - 1) + 1}, "
          f"per level {done.max() / (cols - 1 + 2 * (rows - 1) + 1):.2f} us")
    print("  detect (ready - last dep published) us: mean %.2f p50 %.2f" % (det.mean(), np.median(det)))
    for i, name in enumerate(["wait->ready", "ready->BRS", "BRS->walk", "walk->published"]):
        d = (tr[:, :, i + 1] - tr[:, :, i]).ravel()
        print("  %-16s mean %.3f us p50 %.3f p90 %.3f" % (name, d.mean(), np.median(d), np.percentile(d, 90)))
    # the chain: from the last published block back through the dependency published last
    v, h = np.unravel_index(np.argmax(done), done.shape)
    links = []
    while True:
        cands = [(v, h - 1), (v - 1, h), (v - 1, h + 1)]
        cands = [(a_, b_) for a_, b_ in cands if a_ >= 0 and 0 <= b_ < cols]
        if not cands:
            break
        pv, ph = max(cands, key=lambda x: done[x])
        links.append((tr[v, h, 1] - done[pv, ph], tr[v, h, 4] - tr[v, h, 1], tr[v, h, 0] - done[pv, ph]))
        v, h = pv, ph
    L = np.array(links)
    print("  chain: %d links, detect %.2f us, work %.2f us per link; wait start after dep done: %.0f%% of links (mean %.2f us)"
          % (len(L), L[:, 0].mean(), L[:, 1].mean(), 100 * (L[:, 2] > 0).mean(), L[:, 2][L[:, 2] > 0].mean() if (L[:, 2] > 0).any() else 0))
