"""One interface over the two implementations the tests compare:

  PortBackend  — the CPU oracle restatement (oracle/liboracle.so), test-only;
  GpuBackend   — the product: the CUDA path through the C ABI
                 (paper_1002_1168_b200), used only by -m gpu tests.

Both return plain tuples / numpy arrays so the same assertions run on either.
"""
import numpy as np

import oracle


class PortBackend:
    name = "port"

    def __init__(self):
        self.o = oracle.Oracle("port")

    def run_sequence(self, algo, luma, alpha, bs, S, halfpel=0, ref_distance=2, bt=0, max_iter=4, step=2, eps=0.5, theta=2.0):
        cfg = oracle.make_cfg(algo=algo, search_range=S, block_size=bs, halfpel=halfpel, ref_distance=ref_distance, boundary_temporal=bt, max_iterations=max_iter, step=step, epsilon=eps, theta=theta)
        return self.o.run_sequence(cfg, luma, alpha)

    def block_search(self, algo, cur, ref, x0, y0, size, S):
        mv, cmp, cost = self.o.block_search(algo, cur, ref, x0, y0, size, S)
        return tuple(mv), cmp

    def brs_select(self, cur, ref, ca, ra, x0, y0, size, btype, cands, S, bt):
        mv, kinds = self.o.brs_select(cur, ref, ca, ra, x0, y0, size, btype, cands, S, bt)
        return tuple(mv), list(kinds)

    def prs_refine(self, cur, ref, x0, y0, size, d0, S, step=2, max_iter=4):
        mv, dpd, log = self.o.prs_refine(cur, ref, x0, y0, size, d0, S, step=step, max_iter=max_iter)
        return tuple(mv), dpd, list(log)

    def prs_update(self, cur, ref, x, y, d):
        return self.o.prs_update(cur, ref, x, y, d)

    def sad_texture_q4(self, cur, ref, x0, y0, size, dx, dy):
        return int(round(self.o.sad_texture(cur, ref, x0, y0, size, dx, dy) * 4))

    def sad_shape(self, ca, ra, x0, y0, size, dx, dy):
        return self.o.sad_shape(ca, ra, x0, y0, size, dx, dy)

    def predict(self, ref, mv, types, bs):
        return self.o.predict_frame(ref, mv, types, bs)

    def classify(self, alpha, bs):
        return self.o.classify(alpha, bs)

    def sse(self, a, b):
        return int(((a.astype(np.int64) - b.astype(np.int64)) ** 2).sum())


class GpuBackend:
    name = "gpu"

    def __init__(self):
        import paper_1002_1168_b200 as me

        self.me = me

    def run_sequence(self, algo, luma, alpha, bs, S, halfpel=0, ref_distance=2, bt=0, max_iter=4, step=2, eps=0.5, theta=2.0):
        me = self.me
        cfg = me.BatchConfig(algo=me.Algo(algo), search=me.SearchConfig(search_range=S, block_size=bs, ref_distance=ref_distance, halfpel=bool(halfpel)), prs=me.PrsConfig(epsilon=eps, theta=theta, max_iterations=max_iter, step=step), boundary_temporal=me.BoundaryTemporal(bt))
        recs, stats = me.run_sequences(cfg, luma[None], None if alpha is None else alpha[None])
        return recs[0], stats[0]

    def block_search(self, algo, cur, ref, x0, y0, size, S):
        me = self.me
        st = me.SearchStats()
        fn = [me.full_search, me.tss_search, me.fss_search, me.ds_search][algo]
        mv = fn(cur, ref, me.BlockRect(x0, y0, size), me.SearchConfig(search_range=S, block_size=size), st)
        return tuple(mv), st.block_comparisons

    def brs_select(self, cur, ref, ca, ra, x0, y0, size, btype, cands, S, bt):
        me = self.me
        log = []
        cs = me.CandidateSet(tuple(cands[0:2]), tuple(cands[2:4]), tuple(cands[4:6]), tuple(cands[6:8]))
        mv = me.brs_select(cur, ref, ca, ra, me.BlockRect(x0, y0, size), me.BlockType(btype), cs, me.SearchConfig(search_range=S, block_size=size), me.EstimateOptions(me.BoundaryTemporal(bt), log), me.SearchStats())
        return tuple(mv), [int(e.kind) for e in log]

    def prs_refine(self, cur, ref, x0, y0, size, d0, S, step=2, max_iter=4):
        me = self.me
        st = me.SearchStats()
        log = []
        mv = me.prs_refine(cur, ref, me.BlockRect(x0, y0, size), tuple(d0), me.SearchConfig(search_range=S, block_size=size), me.PrsConfig(step=step, max_iterations=max_iter), st, log)
        return tuple(mv), st.dpd_refinement_steps, [int(round(v * 4)) for v in log]

    def prs_update(self, cur, ref, x, y, d):
        return self.me.prs_update(cur, ref, x, y, tuple(d), self.me.PrsConfig())

    def sad_texture_q4(self, cur, ref, x0, y0, size, dx, dy):
        return int(round(self.me.sad_texture(cur, ref, self.me.BlockRect(x0, y0, size), (dx, dy)) * 4))

    def sad_shape(self, ca, ra, x0, y0, size, dx, dy):
        return self.me.sad_shape(ca, ra, self.me.BlockRect(x0, y0, size), (dx, dy))

    def predict(self, ref, mv, types, bs):
        me = self.me
        h, w = ref.shape
        f = me.MotionField(w // bs, h // bs, bs, vectors=np.ascontiguousarray(mv, np.int32).reshape(-1, 2), types=None if types is None else np.ascontiguousarray(types, np.uint8))
        return me.predict_frame(ref, f, me.SearchConfig(block_size=bs))

    def classify(self, alpha, bs):
        return self.me.classify_blocks(alpha, bs)

    def sse(self, a, b):
        p = self.me.psnr(a, b)
        return int(round(p.mse * a.size))
