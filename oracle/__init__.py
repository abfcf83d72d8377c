"""TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA path.

Two backends with one interface:
  * ``Oracle("port")``       the plain-C restatement (oracle/me_oracle.c ->
                             oracle/liboracle.so), no dependency on the
                             reference at run time;
  * ``Oracle("reference")``  the UNMODIFIED reference sources compiled by
                             oracle/Makefile into oracle/_ref/libme_ref.so,
                             driven by oracle/ref_driver.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs
may import this package; the product (paper_1002_1168_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libme_ref.so")
REF_SRC = "/root/reference/proj"

ME_OK = 0


def build(ref: bool = True, quiet: bool = True):
    """Compiles the restatement (always) and oracle/_ref (when the reference
    sources are present, i.e. in the build container)."""
    target = ["all"]
    if ref and os.path.isdir(REF_SRC):
        target = ["ref"]
    out = subprocess.run(["make", "-C", HERE] + target, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


def _rec_dtype():
    return np.dtype([("dx", "<i2"), ("dy", "<i2"), ("cost_q4", "<u4"), ("comparisons", "<u2"), ("dpd_steps", "<u2"), ("iterations", "u1"), ("type", "u1"), ("reserved", "<u2")])


def _stats_dtype():
    return np.dtype([(n, "<i8") for n in ("block_comparisons", "dpd_refinement_steps", "blocks_opaque", "blocks_boundary", "blocks_transparent", "sse")])


class _Cfg(C.Structure):
    _fields_ = [("algo", C.c_int32), ("search_range", C.c_int32), ("block_size", C.c_int32), ("ref_distance", C.c_int32), ("halfpel", C.c_int32), ("max_iterations", C.c_int32), ("step", C.c_int32), ("boundary_temporal", C.c_int32), ("epsilon", C.c_double), ("theta", C.c_double)]


def make_cfg(algo=4, search_range=16, block_size=8, ref_distance=2, halfpel=0, max_iterations=4, step=2, boundary_temporal=0, epsilon=0.5, theta=2.0):
    return _Cfg(algo, search_range, block_size, ref_distance, halfpel, max_iterations, step, boundary_temporal, epsilon, theta)


def _vp(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.L = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        getattr(self.L, self.p + "last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.L, self.p + name)

    def _chk(self, rc):
        if rc != ME_OK:
            raise OracleError(rc, self._f("last_error")().decode())

    # -- sequences ---------------------------------------------------------
    def run_sequence(self, cfg: _Cfg, luma: np.ndarray, alpha=None, want_pred=False):
        luma = np.ascontiguousarray(luma, np.uint8)
        F, H, W = luma.shape
        if alpha is not None:
            alpha = np.ascontiguousarray(alpha, np.uint8)
        pairs = F - cfg.ref_distance
        bs = cfg.block_size
        recs = np.zeros((pairs, H // bs, W // bs), _rec_dtype())
        stats = np.zeros(pairs, _stats_dtype())
        pred = np.zeros((pairs, H, W), np.uint8) if want_pred else None
        self._chk(self._f("run_sequence")(C.byref(cfg), F, W, H, _vp(luma), _vp(alpha), _vp(recs), _vp(stats), _vp(pred)))
        return (recs, stats, pred) if want_pred else (recs, stats)

    def estimate_field(self, cfg: _Cfg, cur, ref, ca=None, ra=None, prev_mv=None):
        """One pair (port only): orc_estimate_field with an optional previous field."""
        assert self.kind == "port"
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        bs = cfg.block_size
        cols, rows = W // bs, H // bs
        recs = np.zeros(cols * rows, _rec_dtype())
        st = np.zeros(1, _stats_dtype())
        pm = None if prev_mv is None else np.ascontiguousarray(prev_mv, np.int32)
        self._chk(self._f("estimate_field")(C.byref(cfg), W, H, _vp(cur), _vp(ref), _vp(ca), _vp(ra), _vp(pm), cols, rows, _vp(recs), _vp(st)))
        return recs, st[0]

    # -- per block ---------------------------------------------------------
    def block_search(self, algo, cur, ref, x0, y0, size, rng):
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        mv = (C.c_int32 * 2)()
        cmp = C.c_int64()
        cost = C.c_uint32()
        self._chk(self._f("block_search")(algo, W, H, _vp(cur), _vp(ref), x0, y0, size, rng, mv, C.byref(cmp), C.byref(cost)))
        return (mv[0], mv[1]), cmp.value, cost.value

    def brs_select(self, cur, ref, ca, ra, x0, y0, size, btype, cands, rng, bt=0):
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        cd = (C.c_int32 * 8)(*[int(v) for v in cands])
        mv = (C.c_int32 * 2)()
        kinds = (C.c_uint8 * 4)()
        if self.kind == "port":
            scores = (C.c_uint32 * 4)()
            self._chk(self._f("brs_select")(W, H, _vp(cur), _vp(ref), _vp(ca), _vp(ra), x0, y0, size, btype, cd, rng, bt, mv, kinds, scores))
        else:
            cmp = C.c_int64()
            self._chk(self._f("brs_select")(W, H, _vp(cur), _vp(ref), _vp(ca), _vp(ra), x0, y0, size, btype, cd, rng, bt, mv, kinds, C.byref(cmp)))
        return (mv[0], mv[1]), list(kinds)

    def prs_refine(self, cur, ref, x0, y0, size, d0, rng, eps=0.5, theta=2.0, max_iter=4, step=2):
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        d = (C.c_int32 * 2)(*d0)
        mv = (C.c_int32 * 2)()
        dpd = C.c_int64()
        log = (C.c_uint32 * 256)()
        n = C.c_int()
        f = self._f("prs_refine")
        f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._chk(f(W, H, _vp(cur), _vp(ref), x0, y0, size, d, rng, eps, theta, max_iter, step, mv, C.byref(dpd), log, C.byref(n)))
        return (mv[0], mv[1]), dpd.value, [log[i] for i in range(n.value)]

    def prs_update(self, cur, ref, x, y, d, eps=0.5, theta=2.0):
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        dd = (C.c_int32 * 2)(*d)
        out = (C.c_double * 2)()
        f = self._f("prs_update")
        f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        rc = f(W, H, _vp(cur), _vp(ref), x, y, dd, eps, theta, out)
        if self.kind != "port":
            self._chk(rc)
        return out[0], out[1]

    def sad_texture(self, cur, ref, x0, y0, size, dx, dy):
        cur, ref = np.ascontiguousarray(cur), np.ascontiguousarray(ref)
        H, W = cur.shape
        if self.kind == "port":
            f = self._f("sad_texture")
            f.restype = C.c_double
            return f(W, H, _vp(cur), _vp(ref), x0, y0, size, dx, dy)
        out = C.c_double()
        self._chk(self._f("sad_texture")(W, H, _vp(cur), _vp(ref), x0, y0, size, dx, dy, C.byref(out)))
        return out.value

    def sad_shape(self, ca, ra, x0, y0, size, dx, dy):
        ca, ra = np.ascontiguousarray(ca), np.ascontiguousarray(ra)
        H, W = ca.shape
        out = C.c_int64()
        self._chk(self._f("sad_shape")(W, H, _vp(ca), _vp(ra), x0, y0, size, dx, dy, C.byref(out)))
        return out.value

    def classify(self, alpha, size, W=None, H=None):
        if alpha is not None:
            alpha = np.ascontiguousarray(alpha)
            H, W = alpha.shape
        out = np.zeros((H // size) * (W // size), np.uint8)
        self._chk(self._f("classify")(W, H, _vp(alpha), size, _vp(out)))
        return out

    def binarize(self, gray, thr=128):
        gray = np.ascontiguousarray(gray)
        H, W = gray.shape
        out = np.zeros_like(gray)
        self._f("binarize")(W, H, _vp(gray), thr, _vp(out))
        return out

    def predict_frame(self, ref, mv, types, bs):
        ref = np.ascontiguousarray(ref)
        H, W = ref.shape
        mv = np.ascontiguousarray(mv, np.int32)
        types = None if types is None else np.ascontiguousarray(types, np.uint8)
        out = np.zeros_like(ref)
        self._chk(self._f("predict_frame")(W, H, _vp(ref), _vp(mv), _vp(types), bs, _vp(out)))
        return out

    # -- timing (CPU baseline) -------------------------------------------------
    def time_sequences(self, cfg, luma, alpha, threads):
        """n_seq sequences ([n_seq, F, H, W]) on `threads` host threads."""
        n_seq, F, H, W = luma.shape
        if self.kind == "port":
            pairs = F - cfg.ref_distance
            recs = np.zeros((n_seq, pairs, H // cfg.block_size, W // cfg.block_size), _rec_dtype())
            stats = np.zeros((n_seq, pairs), _stats_dtype())
            self._chk(self._f("run_sequences_threaded")(C.byref(cfg), n_seq, F, W, H, _vp(luma), _vp(alpha), _vp(recs), _vp(stats), threads))
            return int(stats["block_comparisons"].sum())
        cs = C.c_int64()
        self._chk(self._f("time_sequences")(C.byref(cfg), n_seq, F, W, H, _vp(luma), _vp(alpha), threads, C.byref(cs)))
        return cs.value

    def time_pairs(self, cfg, luma, alpha, first_pair, n_pairs, threads):
        F, H, W = luma.shape
        if self.kind == "port":
            recs = np.zeros((n_pairs, H // cfg.block_size, W // cfg.block_size), _rec_dtype())
            stats = np.zeros(n_pairs, _stats_dtype())
            self._chk(self._f("run_pairs_threaded")(C.byref(cfg), F, W, H, _vp(luma), _vp(alpha), first_pair, n_pairs, _vp(recs), _vp(stats), threads))
            return int(stats["block_comparisons"].sum())
        cs = C.c_int64()
        self._chk(self._f("time_pairs")(C.byref(cfg), F, W, H, _vp(luma), _vp(alpha), first_pair, n_pairs, threads, C.byref(cs)))
        return cs.value

    def time_blocks(self, cfg, cur, ref, block_xy, threads):
        """Block searches on an explicit (x0, y0) list; returns total comparisons."""
        H, W = cur.shape
        xy = np.ascontiguousarray(block_xy, np.int32)
        n = xy.shape[0]
        if self.kind == "port":
            mv = np.zeros((n, 2), np.int32)
            cmp = np.zeros(n, np.int64)
            self._f("search_blocks")(C.byref(cfg), W, H, _vp(cur), _vp(ref), _vp(xy), n, threads, _vp(mv), _vp(cmp))
            return int(cmp.sum())
        cmp = C.c_int64()
        self._chk(self._f("time_blocks")(C.byref(cfg), W, H, _vp(cur), _vp(ref), _vp(xy), n, threads, C.byref(cmp)))
        return cmp.value

    def run_experiment(self, path, fmt, W, H, mask_pattern, algos, cfg: _Cfg, block_size_auto=True, frame_limit=0, csv_path=None, dump_dir=None):
        """The reference's own run_experiment (bench.cpp:120-227) on a sequence
        file (reference build only).  Returns the AlgoSummary values per algo
        (10 doubles, NaN for absent optionals); the CSV goes to csv_path."""
        if self.kind != "reference":
            raise OracleError(1, "run_experiment needs the reference build")
        a = (C.c_int * len(algos))(*algos)
        out = np.zeros((len(algos), 10), np.float64)
        enc = lambda s: None if s is None else s.encode()
        self._chk(self._f("run_experiment")(enc(path), fmt, W, H, enc(mask_pattern), a, len(algos), C.byref(cfg),
                                            int(block_size_auto), frame_limit, enc(csv_path), enc(dump_dir), _vp(out)))
        return out


# ---------------------------------------------------------------------------
# Input generation for the reference arm (oracle/ref_synth_glue.cpp): the
# product's host generator compiled into oracle/_ref/libme_ref.so, so the
# reference arm never loads libme_b200.so.  Same bytes as
# paper_1002_1168_b200.synth (checked by tests/test_synth.py).


class SynthParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("frames", C.c_int32), ("seed", C.c_uint64),
        ("blur_sigma_q8", C.c_int32), ("bg_jitter", C.c_int32), ("bg_drift_q8", C.c_int32 * 2),
        ("n_objects", C.c_int32), ("obj_min", C.c_int32), ("obj_max", C.c_int32),
        ("obj_w", C.c_int32 * 4), ("obj_h", C.c_int32 * 4), ("obj_v", (C.c_int32 * 2) * 4),
        ("vel_fixed", C.c_int32), ("vmax", C.c_int32), ("shapes", C.c_int32), ("noise_sigma_q8", C.c_int32),
    ]


_REF_HANDLE = None


def _ref_lib():
    global _REF_HANDLE
    if _REF_HANDLE is None:
        _REF_HANDLE = C.CDLL(REF_LIB)
        _REF_HANDLE.ref_synth_last_error.restype = C.c_char_p
    return _REF_HANDLE


def synth_preset(config_id: int, seed: int, frames=None) -> SynthParams:
    L = _ref_lib()
    p = SynthParams()
    if L.ref_synth_preset(int(config_id), C.c_uint64(seed), C.byref(p)) != ME_OK:
        raise OracleError(1, L.ref_synth_last_error().decode())
    if frames:
        p.frames = int(frames)
    return p


def synth_generate(p: SynthParams, luma=None, alpha=None):
    shape = (p.frames, p.height, p.width)
    luma = np.empty(shape, np.uint8) if luma is None else luma
    alpha = np.empty(shape, np.uint8) if alpha is None else alpha
    L = _ref_lib()
    if L.ref_synth(C.byref(p), _vp(luma), _vp(alpha)) != ME_OK:
        raise OracleError(1, L.ref_synth_last_error().decode())
    return luma, alpha


def synth_batch(config_id: int, n_seq: int, base_seed: int, frames=None, threads: int = 8):
    """n_seq sequences with seed = base + i ([n_seq, F, H, W] luma, alpha)."""
    from concurrent.futures import ThreadPoolExecutor

    p0 = synth_preset(config_id, base_seed, frames)
    shape = (n_seq, p0.frames, p0.height, p0.width)
    luma, alpha = np.empty(shape, np.uint8), np.empty(shape, np.uint8)

    def one(i):
        synth_generate(synth_preset(config_id, base_seed + i, frames), luma[i], alpha[i])

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(one, range(n_seq)))
    return luma, alpha


def time_sequences_digest(cfg: _Cfg, luma, alpha, threads: int):
    """The reference's own estimate_field + predict_frame + psnr loop over
    n_seq sequences on `threads` host threads; returns the per-sequence result
    digests (uint64, see ref_driver.cpp Digest)."""
    n_seq, F, H, W = luma.shape
    dig = np.zeros(n_seq, np.uint64)
    cs = C.c_int64()
    L = _ref_lib()
    L.ref_last_error.restype = C.c_char_p
    rc = L.ref_time_sequences_digest(C.byref(cfg), n_seq, F, W, H, _vp(luma), _vp(alpha), threads, C.byref(cs), _vp(dig))
    if rc != ME_OK:
        raise OracleError(rc, L.ref_last_error().decode())
    return dig


def digest_records(recs, stats, W: int, H: int) -> np.ndarray:
    """The same digest from record/stat arrays ([n_seq, pairs, rows, cols] of
    the record dtype, [n_seq, pairs] of the stats dtype), e.g. the CUDA path's."""
    n_seq, pairs, rows, cols = recs.shape
    nb = rows * cols
    dx = recs["dx"].astype(np.int64).astype(np.uint64).reshape(n_seq, pairs * nb)
    dy = recs["dy"].astype(np.int64).astype(np.uint64).reshape(n_seq, pairs * nb)
    w = (2 * np.arange(pairs * nb, dtype=np.uint64) + np.uint64(1))
    with np.errstate(over="ignore"):
        v = ((dx * np.uint64(0x9E37) + dy * np.uint64(0x7F4B) + np.uint64(1)) * w[None, :]).sum(axis=1, dtype=np.uint64)
        st = stats
        s = (st["block_comparisons"].astype(np.uint64) * np.uint64(1000003) + st["dpd_refinement_steps"].astype(np.uint64) * np.uint64(7919)
             + st["blocks_opaque"].astype(np.uint64) * np.uint64(131) + st["blocks_boundary"].astype(np.uint64) * np.uint64(137)
             + st["blocks_transparent"].astype(np.uint64) * np.uint64(139) + st["sse"].astype(np.uint64) * np.uint64(17))
        v = v + s.sum(axis=1, dtype=np.uint64)
    return v
