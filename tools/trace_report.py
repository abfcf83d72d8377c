import numpy as np, sys
for name in ("cfg2", "cfg4"):
    try: raw = open(f"gpurun_out/trace_{name}.bin","rb").read()
    except OSError: continue
    n = len(raw) // 40
    tr = np.frombuffer(raw[:n*32], np.uint64).reshape(n, 4).astype(np.int64)
    lst = np.frombuffer(raw[n*32:], np.uint32).reshape(n, 2)
    valid = tr[:,0] > 0
    tr = tr[valid]; lst = lst[valid]
    t0 = tr[:,0].min()
    claim = (tr[:,0]-t0)/1e3; deps=(tr[:,1]-t0)/1e3; done=(tr[:,2]-t0)/1e3
    h = lst[:,0] & 0xFFFF; v = (lst[:,0]>>16)&0x7FFF; p = lst[:,1]&0xFFFF
    step = h + 2*v + p
    print(name, "tasks", len(tr), "span us %.1f" % done.max())
    print("  wait us: mean %.2f p50 %.2f p90 %.2f" % ((deps-claim).mean(), np.median(deps-claim), np.percentile(deps-claim,90)))
    print("  work us: mean %.2f p50 %.2f p90 %.2f max %.2f" % ((done-deps).mean(), np.median(done-deps), np.percentile(done-deps,90), (done-deps).max()))
    st = np.unique(step)
    md = np.array([done[step==s].max() for s in st])
    print("  per-step increments mean %.2f" % np.diff(md).mean())
