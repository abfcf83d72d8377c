import numpy as np, sys
sys.path.insert(0, '.')
import oracle, paper_1002_1168_b200 as me
port = oracle.Oracle("port")
rng = np.random.default_rng(5)
cur = rng.integers(0, 256, (64, 64), dtype=np.uint8); ref = np.roll(cur, (1, 2), (0, 1))
for algo, fn in ((1, me.tss_search), (2, me.fss_search), (3, me.ds_search)):
    st = me.SearchStats()
    r = me.block_grid(64, 64, 16)[5]
    mv = fn(cur, ref, r, me.SearchConfig(search_range=16, block_size=16), st)
    print(algo, mv, st.block_comparisons, port.block_search(algo, cur, ref, r.x0, r.y0, 16, 16)[:2], flush=True)
