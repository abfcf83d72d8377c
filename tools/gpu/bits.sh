cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bits
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/bits/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/bits/pytest.log
cat > /tmp/bt.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import batch as B, synth, _lib
import ctypes as C
luma, alpha = synth.config4_batch_dev(256, 20260000, 30)
bits, binary = B.pack_mask_dev(alpha)
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
recs = torch.empty((256, 28, 36, 44, 16), dtype=torch.uint8, device='cuda'); stats = torch.empty((256, 28, 48), dtype=torch.uint8, device='cuda')
lib = me.lib(); cx = _lib.ctx(0); st = (C.c_float*4)()
for name, f in (("bytes", lambda: B.run_sequences_dev(cfg, luma, alpha, recs, stats)), ("bits", lambda: B.run_sequences_bits_dev(cfg, luma, bits, recs, stats))):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): f()
    e1.record(); torch.cuda.synchronize()
    _lib.check(lib.me_b200_ctx_set_profiling(cx, 1)); f(); _lib.check(lib.me_b200_ctx_stage_ms(cx, st, 4)); _lib.check(lib.me_b200_ctx_set_profiling(cx, 0))
    print(name, e0.elapsed_time(e1) / 50, [round(x, 4) for x in st])
PY
python /tmp/bt.py
