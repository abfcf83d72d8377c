"""Streaming I/O vs whole-file loading for a sequence file (config 3:
1920x1088 x 60 frames I420, masks as PGM files): seconds for
(a) read every frame, then one run_sequences call, and
(b) seqio.estimate_stream (reader thread + pinned slots + copy stream),
both through the page cache (the file is read once beforehand)."""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import seqio, synth  # noqa: E402

luma, alpha = synth.config_sequence(3, 20260000)
d = tempfile.mkdtemp()
path = os.path.join(d, "cfg3.yuv")
seqio.write_i420(path, luma)
for i in range(luma.shape[0]):
    seqio.write_gray_pgm(alpha[i], os.path.join(d, f"m_{i:03d}.pgm"))
src = seqio.open_sequence(path, luma.shape[2], luma.shape[1])
masks = seqio.MaskSource(pattern=os.path.join(d, "m_%03d.pgm"))
algo = sys.argv[1] if len(sys.argv) > 1 else "PA"
cfg = me.BatchConfig(algo=me.Algo[algo], search=me.SearchConfig(search_range=32, block_size=8 if algo == "PA" else 16))
seqio.read_frames(src)  # warm the page cache
for rep in range(3):
    t = time.perf_counter()
    l = seqio.stream_frames(src)
    a = seqio.read_masks(masks, src.frame_count, src.width, src.height)
    r1, s1 = me.run_sequences(cfg, l[None], a[None])
    ta = time.perf_counter() - t
    res = {}
    for chunk in (4, 8, 16):
        t = time.perf_counter()
        r2, s2 = seqio.estimate_stream(src, cfg, masks, chunk=chunk)
        res[chunk] = round(time.perf_counter() - t, 4)
        assert np.array_equal(r2, r1[0]) and np.array_equal(s2, s1[0])
    print(f"{algo}: whole file then estimate {ta:.4f} s; streamed by chunk size {res} s (results identical)", flush=True)
