"""Analyse a PA wavefront trace (tuning field pa_trace_path, set with
paper_1002_1168_b200._lib.set_tuning(pa_trace_path=...)): per list entry
{claim, deps ready, done, smid} (globaltimer ns) followed by the list.
usage: trace_report.py TRACE.bin COLS ROWS PAIRS"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
cols, rows, pairs = (int(x) for x in sys.argv[2:5])
n = len(raw) // 40
tr = np.frombuffer(raw[: n * 32], np.uint64).reshape(n, 4).astype(np.int64)
lst = np.frombuffer(raw[n * 32:], np.uint32).reshape(n, 2)
valid = tr[:, 0] > 0
tr, lst = tr[valid], lst[valid]
t0 = tr[:, 0].min()
claim, ready, done = ((tr[:, i] - t0) / 1e3 for i in range(3))
h = (lst[:, 0] & 0xFFFF).astype(np.int64)
v = ((lst[:, 0] >> 16) & 0x7FFF).astype(np.int64)
p = (lst[:, 1] & 0xFFFF).astype(np.int64)
seq = (lst[:, 1] >> 16).astype(np.int64)
nseq = seq.max() + 1
step = h + 2 * v + p
grid = np.full((nseq, pairs, rows, cols), -1e9)
grid[seq, p, v, h] = done
def dep(s, pp, vv, hh, ok):
    out = np.full(len(s), -1e9)
    out[ok] = grid[s[ok], pp[ok], vv[ok], hh[ok]]
    return out
dA = dep(seq, p, v, h - 1, h > 0)
dB = dep(seq, p, v - 1, h, v > 0)
dC = dep(seq, p, v - 1, h + 1, (v > 0) & (h + 1 < cols))
dT = dep(seq, p - 1, v, h, p > 0)
dmax = np.maximum.reduce([dA, dB, dC, dT])
has = dmax > -1e8
print("tasks", len(tr), "span us %.1f" % done.max(), "steps", step.max() + 1)
cyc = np.stack([(tr[:, 3] >> (16 * i)) & 0xFFFF for i in range(4)], 1).astype(np.float64)
for i, name in enumerate(["ready->staged", "staged->brs", "brs->walked", "walked->published"]):
    print("cycles %-18s mean %7.0f p50 %7.0f p90 %7.0f" % (name, cyc[:, i].mean(), *np.percentile(cyc[:, i], [50, 90])))
bnd = (lst[:, 0] >> 31).astype(bool)
for flag, name in ((False, "opaque"), (True, "boundary")):
    m = bnd == flag
    if m.any():
        print("  %-8s blocks %6d  ready->staged mean %6.0f  staged->brs %6.0f  brs->walked %6.0f" % (name, m.sum(), cyc[m, 0].mean(), cyc[m, 1].mean(), cyc[m, 2].mean()))
print("work (ready->done) us: mean %.2f p50 %.2f p90 %.2f p99 %.2f" % ((done - ready).mean(), *np.percentile(done - ready, [50, 90, 99])))
print("claim->ready us:       mean %.2f p50 %.2f p90 %.2f" % ((ready - claim).mean(), *np.percentile(ready - claim, [50, 90])))
late = ready[has] - dmax[has]
print("detect (ready - last dep done) us: mean %.2f p50 %.2f p90 %.2f" % (late.mean(), *np.percentile(late, [50, 90])))
slack = claim[has] - dmax[has]
print("claim - last dep done us: mean %.2f p50 %.2f (negative = claimed before its deps finished: %.0f%%)" % (slack.mean(), np.median(slack), 100 * (slack < 0).mean()))
st = np.unique(step)
md = np.array([done[step == s].max() for s in st])
mc = np.array([claim[step == s].min() for s in st])
print("per-step: last-done increments mean %.2f us; first-claim increments mean %.2f us" % (np.diff(md).mean(), np.diff(mc).mean()))
cnt = np.array([(step == s).sum() for s in st])
print("items per step: min %d mean %.0f max %d" % (cnt.min(), cnt.mean(), cnt.max()))
for q in (10, 50, 90):
    i = int(len(st) * q / 100)
    print("  step %d: items %d, claim %.1f..%.1f us, done max %.1f us" % (st[i], cnt[i], claim[step == st[i]].min(), claim[step == st[i]].max(), md[i]))
# Critical chain: walk back from the last-published block through the dependency
# that finished last, splitting the span into per-block work (start -> done, start
# = max(claim, last dep done)) and claim waits (claim later than the last dep).
idx = np.full((nseq, pairs, rows, cols), -1, np.int64)
idx[seq, p, v, h] = np.arange(len(done))
i = int(np.argmax(done))
chain = []
while True:
    chain.append(i)
    cands = []
    s_, p_, v_, h_ = seq[i], p[i], v[i], h[i]
    for (pp, vv, hh) in ((p_, v_, h_ - 1), (p_, v_ - 1, h_), (p_, v_ - 1, h_ + 1), (p_ - 1, v_, h_)):
        if pp >= 0 and vv >= 0 and 0 <= hh < cols and idx[s_, pp, vv, hh] >= 0:
            cands.append(idx[s_, pp, vv, hh])
    if not cands:
        break
    j = max(cands, key=lambda k: done[k])
    if done[j] < claim[i] - 50:  # claimed well after this dep finished: the chain goes through the claim
        break
    i = j
chain = chain[::-1]
ch = np.array(chain)
st0 = np.maximum(claim[ch], np.r_[claim[ch[0]], done[ch[:-1]]])
work = done[ch] - st0
cw = np.maximum(0, claim[ch] - np.r_[claim[ch[0]], done[ch[:-1]]])
print("critical chain: %d blocks, first claim %.1f us, end %.1f us; work %.1f us (mean %.2f/block), claim waits %.1f us"
      % (len(ch), claim[ch[0]], done[ch[-1]], work.sum(), work.mean(), cw[1:].sum()))
print("  chain ready->done mean %.2f us, detect (ready - dep done) mean %.2f us" % ((done[ch] - ready[ch]).mean(), (ready[ch][1:] - done[ch[:-1]]).mean()))
# DAG depth of the traced list (levels)
lev = np.zeros(len(done), np.int64)
order = np.argsort(step, kind="stable")
for k in order:
    m = 0
    s_, p_, v_, h_ = seq[k], p[k], v[k], h[k]
    for (pp, vv, hh) in ((p_, v_, h_ - 1), (p_, v_ - 1, h_), (p_, v_ - 1, h_ + 1), (p_ - 1, v_, h_)):
        if pp >= 0 and vv >= 0 and 0 <= hh < cols:
            j = idx[s_, pp, vv, hh]
            if j >= 0:
                m = max(m, lev[j])
    lev[k] = m + 1
print("DAG depth %d (list steps %d); span / depth = %.2f us per level" % (lev.max(), step.max() + 1, done.max() / lev.max()))
# Per-step profile (every 4th step): items, window of claims, last done, the
# mean claim->ready and ready->done and the mean patch-staging cycles.
if len(sys.argv) > 5 and sys.argv[5] == "steps":
    print("step items claim0 claim1 done1 | claim->ready ready->done staged_cyc brs_cyc walk_cyc")
    for s in st[::2]:
        m = step == s
        print("%4d %6d %7.1f %7.1f %7.1f | %5.2f %5.2f %6.0f %6.0f %6.0f" % (
            s, m.sum(), claim[m].min(), claim[m].max(), done[m].max(), (ready[m] - claim[m]).mean(),
            (done[m] - ready[m]).mean(), cyc[m, 0].mean(), cyc[m, 1].mean(), cyc[m, 2].mean()))
