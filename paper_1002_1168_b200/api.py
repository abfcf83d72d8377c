"""Host-side mirror of the reference's motion-estimation API
(/root/reference/proj/include/me/estimators.hpp, compensation.hpp, metrics.hpp,
frame.hpp), backed by the sm_100a kernels through the C ABI.

Same names, argument meaning and error behaviour as the reference:
``ValueError`` where it throws ``std::invalid_argument``, ``IndexError`` where it
throws ``std::out_of_range``.  Frames and alpha planes are 2-D ``uint8`` numpy
arrays (row-major, pitch == width, the reference's ``me::Plane``); motion
vectors are half-pel ``(dx, dy)`` tuples.

Only trivial integer bookkeeping (window clipping, candidate gathering, config
validation, the final PSNR log10 of a GPU-computed SSE) runs on the host; every
pixel operation runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from ._lib import MeConfig, check, ctx, lib

MV = Tuple[int, int]


class Algo(enum.IntEnum):  # estimators.hpp:29
    ES = 0
    TSS = 1
    FSS = 2
    DS = 3
    PA = 4


def to_string(a: "Algo") -> str:  # estimators.cpp:116-125
    return Algo(a).name


def algo_from_string(name: str) -> Algo:  # estimators.cpp:127-137
    up = name.upper()
    if up == "4SS":
        up = "FSS"
    if up in ("ES", "TSS", "FSS", "DS", "PA"):
        return Algo[up]
    raise ValueError("unknown algorithm: " + name)


class BlockType(enum.IntEnum):  # frame.hpp:71
    Transparent = 0
    Opaque = 1
    Boundary = 2


class BoundaryTemporal(enum.IntEnum):  # estimators.hpp:82
    Texture = 0
    Shape = 1


class ScoreKind(enum.IntEnum):  # estimators.hpp:85
    Texture = 0
    Shape = 1


@dataclass
class SearchConfig:  # estimators.hpp:34-41
    search_range: int = 7
    block_size: int = 16
    ref_distance: int = 2
    halfpel: bool = False

    def validate(self):  # estimators.cpp:139-143
        if self.search_range < 1:
            raise ValueError("search_range must be >= 1")
        if self.block_size not in (8, 16):
            raise ValueError("block_size must be 8 or 16")
        if self.ref_distance < 1:
            raise ValueError("ref_distance must be >= 1")


@dataclass
class PrsConfig:  # estimators.hpp:43-50
    epsilon: float = 0.5
    theta: float = 2.0
    max_iterations: int = 4
    step: int = 2

    def validate(self):  # estimators.cpp:145-150
        if not (self.epsilon > 0.0):
            raise ValueError("epsilon must be > 0")
        if not (self.theta > 0.0):
            raise ValueError("theta must be > 0")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.step not in (1, 2):
            raise ValueError("step must be 1 or 2 half-pels")


@dataclass
class BlockRect:  # frame.hpp:76-82
    x0: int = 0
    y0: int = 0
    size: int = 16
    grid_h: int = 0
    grid_v: int = 0


@dataclass
class ScoreEvent:  # estimators.hpp:88-94
    h: int = 0
    v: int = 0
    type: BlockType = BlockType.Opaque
    candidate: int = 0
    kind: ScoreKind = ScoreKind.Texture


@dataclass
class EstimateOptions:  # estimators.hpp:96-99
    boundary_temporal: BoundaryTemporal = BoundaryTemporal.Texture
    scoring_log: Optional[List[ScoreEvent]] = None


@dataclass
class SearchStats:  # metrics.hpp:40-62
    block_comparisons: int = 0
    dpd_refinement_steps: int = 0
    blocks_opaque: int = 0
    blocks_boundary: int = 0
    blocks_transparent: int = 0
    elapsed_us: int = 0

    def blocks_total(self):
        return self.blocks_opaque + self.blocks_boundary + self.blocks_transparent

    def blocks_estimated(self):
        return self.blocks_opaque + self.blocks_boundary

    def search_points(self):
        return self.block_comparisons + self.dpd_refinement_steps

    def merge(self, o: "SearchStats"):
        self.block_comparisons += o.block_comparisons
        self.dpd_refinement_steps += o.dpd_refinement_steps
        self.blocks_opaque += o.blocks_opaque
        self.blocks_boundary += o.blocks_boundary
        self.blocks_transparent += o.blocks_transparent
        self.elapsed_us += o.elapsed_us


@dataclass
class CandidateSet:  # estimators.hpp:78-83
    a: MV = (0, 0)
    b: MV = (0, 0)
    c: MV = (0, 0)
    t: MV = (0, 0)


@dataclass
class MotionField:  # estimators.hpp:56-73, estimators.cpp:152-159
    cols: int
    rows: int
    block_size: int = 16
    cur_index: int = 0
    ref_index: int = 0
    vectors: np.ndarray = field(default=None)  # [rows*cols, 2] int32 (dx, dy)
    types: np.ndarray = field(default=None)    # [rows*cols] uint8 BlockType

    def __post_init__(self):
        if self.cols <= 0 or self.rows <= 0:
            raise ValueError("empty motion field grid")
        n = self.cols * self.rows
        if self.vectors is None:
            self.vectors = np.zeros((n, 2), np.int32)
        if self.types is None:
            self.types = np.full(n, int(BlockType.Opaque), np.uint8)

    def at(self, h: int, v: int) -> MV:
        dx, dy = self.vectors[v * self.cols + h]
        return int(dx), int(dy)

    def set(self, h: int, v: int, mv: MV):
        self.vectors[v * self.cols + h] = mv

    def type_at(self, h: int, v: int) -> BlockType:
        return BlockType(int(self.types[v * self.cols + h]))

    def __eq__(self, o):
        return (
            isinstance(o, MotionField)
            and (self.cols, self.rows, self.block_size, self.cur_index, self.ref_index)
            == (o.cols, o.rows, o.block_size, o.cur_index, o.ref_index)
            and np.array_equal(self.vectors, o.vectors)
            and np.array_equal(self.types, o.types)
        )


@dataclass
class PsnrResult:  # metrics.hpp:30-37
    mse: float = 0.0
    psnr_db: Optional[float] = None
    psnr_linear: Optional[float] = None

    def infinite(self):
        return self.psnr_db is None


# ---------------------------------------------------------------------------
# helpers


def _plane(a, name="plane") -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint8 or a.ndim != 2:
        raise ValueError(f"{name} must be a 2-D uint8 array")
    return a


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _cfg(algo: int, s: SearchConfig, p: PrsConfig, bt: int = 0) -> MeConfig:
    c = MeConfig()
    c.algo = int(algo)
    c.search_range = s.search_range
    c.block_size = s.block_size
    c.ref_distance = s.ref_distance
    c.halfpel = 1 if s.halfpel else 0
    c.max_iterations = p.max_iterations
    c.step = p.step
    c.boundary_temporal = int(bt)
    c.epsilon = float(p.epsilon)
    c.theta = float(p.theta)
    return c


def check_dimensions(width: int, height: int):  # frame.cpp:34-40
    if width <= 0 or height <= 0:
        raise ValueError("frame dimensions must be positive")
    if width % 16 or height % 16:
        raise ValueError(f"frame dimensions must be multiples of 16, got {width}x{height}")


def block_grid(width: int, height: int, size: int) -> List[BlockRect]:  # frame.cpp:106-119
    if size <= 0 or width % size or height % size:
        raise ValueError(f"block size {size} does not divide {width}x{height}")
    return [BlockRect(h * size, v * size, size, h, v) for v in range(height // size) for h in range(width // size)]


def _window(rect: BlockRect, width: int, height: int, range_pels: int):  # estimators.cpp:41-48
    return (
        max(-2 * range_pels, -2 * rect.x0),
        min(2 * range_pels, 2 * (width - rect.x0 - rect.size)),
        max(-2 * range_pels, -2 * rect.y0),
        min(2 * range_pels, 2 * (height - rect.y0 - rect.size)),
    )


def clip_to_window(v: MV, rect: BlockRect, width: int, height: int, range_pels: int) -> MV:
    """estimators.cpp:161-165 (integer bookkeeping, host)."""
    lo_x, hi_x, lo_y, hi_y = _window(rect, width, height, range_pels)
    return (min(max(v[0], lo_x), hi_x), min(max(v[1], lo_y), hi_y))


# ---------------------------------------------------------------------------
# frame.cpp / metrics.cpp entry points (GPU)


def binarize(gray, threshold: int = 128) -> np.ndarray:  # frame.cpp:50-56
    g = _plane(gray, "gray")
    out = np.empty_like(g)
    check(lib().me_b200_binarize(ctx(), g.shape[1], g.shape[0], _ptr(g), int(threshold), _ptr(out)))
    return out


def classify_block(alpha, rect: BlockRect) -> BlockType:  # frame.cpp:81-104
    if alpha is None:
        return BlockType.Opaque
    a = _plane(alpha, "alpha")
    h, w = a.shape
    if rect.x0 < 0 or rect.y0 < 0 or rect.x0 + rect.size > w or rect.y0 + rect.size > h:
        raise IndexError("block rect outside alpha plane")
    # classify the cropped block as a one-block grid; edge-replicating pad to a
    # multiple of 4 changes neither "any set" nor "all set"
    sub = a[rect.y0 : rect.y0 + rect.size, rect.x0 : rect.x0 + rect.size]
    pad = (-rect.size) % 4
    if pad:
        sub = np.pad(sub, ((0, pad), (0, pad)), mode="edge")
    sub = np.ascontiguousarray(sub)
    return BlockType(int(classify_blocks(sub, sub.shape[0])[0]))


def classify_blocks(alpha, block_size: int) -> np.ndarray:
    """classify_block over the raster block grid (estimators.cpp:410-412)."""
    a = _plane(alpha, "alpha")
    out = np.empty((a.shape[0] // block_size) * (a.shape[1] // block_size), np.uint8)
    check(lib().me_b200_classify_blocks(ctx(), a.shape[1], a.shape[0], _ptr(a), block_size, _ptr(out)))
    return out


def sad_texture(cur, ref, rect: BlockRect, mv: MV) -> float:  # metrics.cpp:43-63
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    out = C.c_uint32()
    check(lib().me_b200_sad_texture(ctx(), c.shape[1], c.shape[0], _ptr(c), _ptr(r), rect.x0, rect.y0, rect.size, int(mv[0]), int(mv[1]), C.byref(out)))
    return out.value / 4.0


def sad_shape(cur_alpha, ref_alpha, rect: BlockRect, mv: MV) -> int:  # metrics.cpp:65-84
    c, r = _plane(cur_alpha), _plane(ref_alpha)
    out = C.c_int64()
    check(lib().me_b200_sad_shape(ctx(), c.shape[1], c.shape[0], _ptr(c), _ptr(r), rect.x0, rect.y0, rect.size, int(mv[0]), int(mv[1]), C.byref(out)))
    return out.value


def block_dpd_aggregate(cur, ref, rect: BlockRect, d: MV) -> float:  # metrics.cpp:90-95
    return sad_texture(cur, ref, rect, (-d[0], -d[1]))


def psnr_from_sse(sse: int, n: int) -> PsnrResult:  # metrics.cpp:117-123
    r = PsnrResult(mse=float(sse) / float(n))
    if sse != 0:
        r.psnr_linear = 255.0 * 255.0 / r.mse
        r.psnr_db = 10.0 * math.log10(r.psnr_linear)
    return r


def psnr(cur, recon) -> PsnrResult:  # metrics.cpp:108-124 (SSE on the GPU)
    a, b = _plane(cur), _plane(recon)
    if a.shape != b.shape:
        raise ValueError("psnr: frame dimensions differ")
    out = C.c_int64()
    check(lib().me_b200_sse(ctx(), a.shape[1], a.shape[0], _ptr(a), _ptr(b), C.byref(out)))
    return psnr_from_sse(out.value, a.size)


def figure_of_merit(psnr_linear: float, s: int, c: float) -> float:  # metrics.cpp:126-131
    if s < 1:
        raise ValueError("figure_of_merit: search range must be >= 1")
    if not (c > 0.0):
        raise ValueError("figure_of_merit: average compared blocks must be > 0")
    window = float(2 * s + 1) * float(2 * s + 1)
    return psnr_linear * window / c


# ---------------------------------------------------------------------------
# estimators.cpp entry points (GPU)


def _require_inside(cur: np.ndarray, rect: BlockRect):  # estimators.cpp:105-110
    h, w = cur.shape
    if rect.x0 < 0 or rect.y0 < 0 or rect.size <= 0 or rect.x0 + rect.size > w or rect.y0 + rect.size > h:
        raise ValueError("block rect outside the frame")


def _block_search(algo: Algo, cur, ref, rect: BlockRect, cfg: SearchConfig, stats: SearchStats) -> MV:
    cfg.validate()
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    _require_inside(c, rect)
    mv = (C.c_int32 * 2)()
    cmp = C.c_int64()
    cost = C.c_uint32()
    check(lib().me_b200_block_search(ctx(), int(algo), c.shape[1], c.shape[0], _ptr(c), _ptr(r), rect.x0, rect.y0, rect.size, cfg.search_range, mv, C.byref(cmp), C.byref(cost)))
    stats.block_comparisons += cmp.value
    return int(mv[0]), int(mv[1])


def full_search(cur, ref, rect, cfg, stats) -> MV:  # estimators.cpp:167-187
    return _block_search(Algo.ES, cur, ref, rect, cfg, stats)


def tss_search(cur, ref, rect, cfg, stats) -> MV:  # estimators.cpp:189-200
    return _block_search(Algo.TSS, cur, ref, rect, cfg, stats)


def fss_search(cur, ref, rect, cfg, stats) -> MV:  # estimators.cpp:202-216
    return _block_search(Algo.FSS, cur, ref, rect, cfg, stats)


def ds_search(cur, ref, rect, cfg, stats) -> MV:  # estimators.cpp:218-236
    return _block_search(Algo.DS, cur, ref, rect, cfg, stats)


def gather_candidates(field_in_progress: MotionField, prev_field: Optional[MotionField], h: int, v: int) -> CandidateSet:
    """estimators.cpp:238-255 (integer bookkeeping, host)."""
    f = field_in_progress
    if h < 0 or v < 0 or h >= f.cols or v >= f.rows:
        raise IndexError("block coordinates outside the motion field grid")
    cs = CandidateSet()
    if h - 1 >= 0:
        cs.a = f.at(h - 1, v)
    if v - 1 >= 0:
        cs.b = f.at(h, v - 1)
    if h + 1 < f.cols and v - 1 >= 0:
        cs.c = f.at(h + 1, v - 1)
    if prev_field is not None:
        if prev_field.cols != f.cols or prev_field.rows != f.rows:
            raise ValueError("previous motion field grid mismatch")
        cs.t = prev_field.at(h, v)
    return cs


def brs_select(cur, ref, cur_alpha, ref_alpha, rect: BlockRect, btype: BlockType, cands: CandidateSet, cfg: SearchConfig, opts: EstimateOptions, stats: SearchStats) -> MV:
    """estimators.cpp:257-301."""
    cfg.validate()
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    _require_inside(c, rect)
    if btype == BlockType.Transparent:
        raise ValueError("candidate selection on a transparent block")
    if btype == BlockType.Boundary and (cur_alpha is None or ref_alpha is None):
        raise ValueError("boundary block requires both alpha planes")
    ca = None if cur_alpha is None else _plane(cur_alpha)
    ra = None if ref_alpha is None else _plane(ref_alpha)
    cd = (C.c_int32 * 8)(*cands.a, *cands.b, *cands.c, *cands.t)
    mv = (C.c_int32 * 2)()
    kinds = (C.c_uint8 * 4)()
    scores = (C.c_uint32 * 4)()
    check(lib().me_b200_brs_select(ctx(), c.shape[1], c.shape[0], _ptr(c), _ptr(r), _ptr(ca), _ptr(ra), rect.x0, rect.y0, rect.size, int(btype), cd, cfg.search_range, int(opts.boundary_temporal), mv, kinds, scores))
    stats.block_comparisons += 4
    if opts.scoring_log is not None:
        for i in range(4):
            opts.scoring_log.append(ScoreEvent(rect.x0 // rect.size, rect.y0 // rect.size, BlockType(btype), i, ScoreKind(kinds[i])))
    return int(mv[0]), int(mv[1])


def prs_update(cur, ref, x: int, y: int, d_i: MV, cfg: PrsConfig):
    """estimators.cpp:303-309 (one pixel, on the GPU); returns (x, y) in pels."""
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    d = (C.c_int32 * 2)(int(d_i[0]), int(d_i[1]))
    out = (C.c_double * 2)()
    check(lib().me_b200_prs_update(ctx(), c.shape[1], c.shape[0], _ptr(c), _ptr(r), int(x), int(y), d, float(cfg.epsilon), float(cfg.theta), out))
    return out[0], out[1]


def prs_refine(cur, ref, rect: BlockRect, d0: MV, scfg: SearchConfig, cfg: PrsConfig, stats: SearchStats, descent_log: Optional[list] = None) -> MV:
    """estimators.cpp:311-382."""
    scfg.validate()
    cfg.validate()
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    _require_inside(c, rect)
    d = (C.c_int32 * 2)(int(d0[0]), int(d0[1]))
    mv = (C.c_int32 * 2)()
    dpd = C.c_int64()
    log = (C.c_uint32 * 64)()
    n = C.c_int()
    check(lib().me_b200_prs_refine(ctx(), c.shape[1], c.shape[0], _ptr(c), _ptr(r), rect.x0, rect.y0, rect.size, d, scfg.search_range, float(cfg.epsilon), float(cfg.theta), int(cfg.max_iterations), int(cfg.step), mv, C.byref(dpd), log, C.byref(n)))
    stats.dpd_refinement_steps += dpd.value
    if descent_log is not None:
        descent_log.extend(log[i] / 4.0 for i in range(n.value))
    return int(mv[0]), int(mv[1])


def estimate_field(algo: Algo, cur, ref, cur_alpha, ref_alpha, prev_field: Optional[MotionField], cfg: SearchConfig, prs: PrsConfig, opts: Optional[EstimateOptions] = None, cur_index: int = 0, ref_index: int = 0, return_records: bool = False):
    """estimators.cpp:384-440: one frame pair on the GPU; returns (MotionField, SearchStats)."""
    opts = opts or EstimateOptions()
    cfg.validate()
    prs.validate()
    c, r = _plane(cur, "cur"), _plane(ref, "ref")
    if c.shape != r.shape:
        raise ValueError("current and reference frame dimensions differ")
    h, w = c.shape
    bs = cfg.block_size
    if w % bs or h % bs:
        raise ValueError(f"block size {bs} does not divide {w}x{h}")
    cols, rows = w // bs, h // bs
    if prev_field is not None and (prev_field.cols != cols or prev_field.rows != rows):
        raise ValueError("previous motion field grid mismatch")
    ca = None if cur_alpha is None else _plane(cur_alpha)
    ra = None if ref_alpha is None else _plane(ref_alpha)
    prev = None if prev_field is None else np.ascontiguousarray(prev_field.vectors, np.int32)
    recs = np.zeros(cols * rows, _lib.rec_dtype())
    st = np.zeros(1, _lib.stats_dtype())
    check(lib().me_b200_estimate_field(ctx(), C.byref(_cfg(algo, cfg, prs, opts.boundary_temporal)), w, h, _ptr(c), _ptr(r), _ptr(ca), _ptr(ra), _ptr(prev), cols, rows, _ptr(recs), _ptr(st)))
    field_ = MotionField(cols, rows, bs, cur_index, ref_index)
    field_.vectors[:, 0] = recs["dx"]
    field_.vectors[:, 1] = recs["dy"]
    field_.types[:] = recs["type"]
    stats = SearchStats(int(st["block_comparisons"][0]), int(st["dpd_refinement_steps"][0]), int(st["blocks_opaque"][0]), int(st["blocks_boundary"][0]), int(st["blocks_transparent"][0]))
    if opts.scoring_log is not None and algo == Algo.PA:
        # the scoring kind is a pure function of (type, candidate, boundary_temporal)
        # (estimators.cpp:277-279); raster order of the estimated blocks
        for i in range(cols * rows):
            t = int(recs["type"][i])
            if t == BlockType.Transparent:
                continue
            for k in range(4):
                shape = t == BlockType.Boundary and (k < 3 or opts.boundary_temporal == BoundaryTemporal.Shape)
                opts.scoring_log.append(ScoreEvent(i % cols, i // cols, BlockType(t), k, ScoreKind(int(shape))))
    if return_records:
        return field_, stats, recs
    return field_, stats


# ---------------------------------------------------------------------------
# compensation.cpp entry points


def predict_frame(ref, field_: MotionField, cfg: SearchConfig, cur=None):
    """compensation.cpp:30-71 (luma).  Returns the predicted luma plane; with
    ``cur`` also the int64 SSE of cur vs the prediction (fused on the GPU)."""
    cfg.validate()
    if field_.block_size != cfg.block_size:
        raise ValueError("motion field block size does not match the configuration")
    r = _plane(ref, "ref")
    if field_.cols * field_.block_size != r.shape[1] or field_.rows * field_.block_size != r.shape[0]:
        raise ValueError("motion field grid does not cover the frame")
    mv = np.ascontiguousarray(field_.vectors, np.int32)
    ty = np.ascontiguousarray(field_.types, np.uint8)
    c = None if cur is None else _plane(cur, "cur")
    out = np.empty_like(r)
    sse = C.c_int64()
    check(lib().me_b200_predict_frame(ctx(), r.shape[1], r.shape[0], _ptr(r), _ptr(mv), _ptr(ty), field_.block_size, _ptr(c), _ptr(out), C.byref(sse)))
    if cur is not None:
        return out, sse.value
    return out


def residual(cur, pred) -> np.ndarray:  # compensation.cpp:73-84 (host utility, off the hot path)
    a, b = _plane(cur), _plane(pred)
    if a.shape != b.shape:
        raise ValueError("residual operands have different dimensions")
    return a.astype(np.int16) - b.astype(np.int16)


def residual_to_gray(r: np.ndarray) -> np.ndarray:  # compensation.cpp:86-94 (visualisation)
    return np.clip(r.astype(np.int32) + 128, 0, 255).astype(np.uint8)
