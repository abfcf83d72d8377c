import sys
import torch
sys.path.insert(0, ".")
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import _lib, batch as B, synth
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
n=int(sys.argv[1]); plain=int(sys.argv[2])
luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
_lib.set_tuning(0, pa_key_plain=plain)
for _ in range(2): B.run_sequences_dev(cfg, luma, alpha)
torch.cuda.synchronize()
