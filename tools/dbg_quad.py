import os
import numpy as np
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import synth
luma, alpha = synth.config4_batch(5, 700, frames=6)
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
recs, stats = me.run_sequences(cfg, luma, alpha)
print("ok", stats.shape)
