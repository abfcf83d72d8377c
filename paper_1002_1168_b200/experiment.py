"""The reference's experiment driver (bench.cpp:120-227, bench.hpp:33-101) on
the batched GPU path.

``run_experiment`` estimates every frame pair of a sequence with ONE batched
call per algorithm (``me_b200_run_sequences``: classify -> wavefront sort ->
search -> fused MC+PSNR SSE, the PA temporal chain inside the call) and turns
the per-pair records and stats into the reference's ``FrameReport`` rows, CSV
(``kCsvHeader`` / ``csv_row``, byte-identical except ``elapsed_us``) and
``AlgoSummary`` (Eq. 6 figure of merit), optionally dumping the reference's
artifacts (``dump_artifacts``: pred/resid PGMs and the vector file).

``elapsed_us`` is the batched call's wall time divided evenly over its pairs
(the reference times each pair's block loop separately).
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import api, seqio
from .api import Algo, BoundaryTemporal, PrsConfig, SearchConfig

CSV_HEADER = "frame,algo,psnr_db,mse,avg_search_points,dpd_steps,n_opaque,n_boundary,n_transparent,elapsed_us"  # bench.cpp:47-49


def fmt_double(v: float) -> str:  # bench.cpp:33-37 ("%.17g")
    return "%.17g" % v


@dataclass
class ExperimentConfig:  # bench.hpp:33-47
    source: seqio.SequenceSource = field(default_factory=seqio.SequenceSource)
    masks: seqio.MaskSource = field(default_factory=seqio.MaskSource)
    algos: List[Algo] = field(default_factory=list)
    search: SearchConfig = field(default_factory=SearchConfig)
    prs: PrsConfig = field(default_factory=PrsConfig)
    boundary_temporal: BoundaryTemporal = BoundaryTemporal.Texture
    block_size_auto: bool = True  # 16 for the block matchers, 8 for PA (bench.cpp:145)
    csv_path: str = ""
    dump_dir: str = ""
    frame_limit: int = 0

    def frames_used(self) -> int:  # bench.cpp:60-63
        if self.frame_limit > 0:
            return min(self.frame_limit, self.source.frame_count)
        return self.source.frame_count

    def validate(self):  # bench.cpp:51-58
        if not self.algos:
            raise ValueError("no algorithm selected")
        self.search.validate()
        self.prs.validate()
        if self.source.frame_count <= 0:
            raise ValueError("sequence has no frames")
        if self.search.ref_distance >= self.frames_used():
            raise ValueError("ref_distance must be smaller than the frame count")


@dataclass
class FrameReport:  # bench.hpp:50-64
    frame: int = 0
    algo: Algo = Algo.ES
    psnr: api.PsnrResult = field(default_factory=api.PsnrResult)
    avg_search_points: Optional[float] = None
    comparisons: int = 0
    dpd_steps: int = 0
    n_opaque: int = 0
    n_boundary: int = 0
    n_transparent: int = 0
    elapsed_us: int = 0

    def blocks_estimated(self) -> int:
        return self.n_opaque + self.n_boundary


@dataclass
class AlgoSummary:  # bench.hpp:67-81
    algo: Algo = Algo.ES
    frame_pairs: int = 0
    mean_mse: float = 0.0
    mean_psnr_db: Optional[float] = None
    psnr_db_of_mean_mse: Optional[float] = None
    mean_psnr_linear: Optional[float] = None
    avg_search_points: float = 0.0
    indicator: Optional[float] = None
    total_comparisons: int = 0
    total_dpd_steps: int = 0
    total_blocks_estimated: int = 0
    total_elapsed_us: int = 0


@dataclass
class ExperimentResult:  # bench.hpp:83-86
    reports: List[FrameReport] = field(default_factory=list)
    summaries: List[AlgoSummary] = field(default_factory=list)


def csv_row(r: FrameReport) -> str:  # bench.cpp:65-74
    return ",".join([
        str(r.frame), api.to_string(r.algo),
        fmt_double(r.psnr.psnr_db) if r.psnr.psnr_db is not None else "inf",
        fmt_double(r.psnr.mse),
        fmt_double(r.avg_search_points) if r.avg_search_points is not None else "nan",
        str(r.dpd_steps), str(r.n_opaque), str(r.n_boundary), str(r.n_transparent), str(r.elapsed_us),
    ])


def algo_search_config(cfg: ExperimentConfig, algo: Algo) -> SearchConfig:
    s = SearchConfig(search_range=cfg.search.search_range, block_size=cfg.search.block_size,
                     ref_distance=cfg.search.ref_distance, halfpel=cfg.search.halfpel)
    if cfg.block_size_auto:  # bench.cpp:145
        s.block_size = 8 if algo == Algo.PA else 16
    return s


def reports_from_stats(algo: Algo, stats: np.ndarray, npix: int, first_frame: int,
                       elapsed_us: Sequence[int]) -> List[FrameReport]:
    """Per-pair FrameReports (bench.cpp:163-184) from me_pair_stats rows (the
    exact per-pair SSE of predict_frame + psnr comes with them)."""
    out = []
    for i, st in enumerate(stats):
        r = FrameReport(frame=first_frame + i, algo=algo)
        r.psnr = api.psnr_from_sse(int(st["sse"]), npix)
        r.comparisons = int(st["block_comparisons"])
        r.dpd_steps = int(st["dpd_refinement_steps"])
        r.n_opaque = int(st["blocks_opaque"])
        r.n_boundary = int(st["blocks_boundary"])
        r.n_transparent = int(st["blocks_transparent"])
        r.elapsed_us = int(elapsed_us[i])
        if r.blocks_estimated() > 0:
            r.avg_search_points = float(r.comparisons) / float(r.blocks_estimated())
        out.append(r)
    return out


def summarize(algo: Algo, reports: Sequence[FrameReport], search_range: int) -> AlgoSummary:
    """AlgoSummary of one algorithm's pairs (bench.cpp:186-217), sums in pair order."""
    s = AlgoSummary(algo=algo)
    mse_sum = db_sum = lin_sum = 0.0
    finite = 0
    for r in reports:
        s.frame_pairs += 1
        mse_sum += r.psnr.mse
        if r.psnr.psnr_db is not None:
            db_sum += r.psnr.psnr_db
            lin_sum += r.psnr.psnr_linear
            finite += 1
        s.total_comparisons += r.comparisons
        s.total_dpd_steps += r.dpd_steps
        s.total_blocks_estimated += r.blocks_estimated()
        s.total_elapsed_us += r.elapsed_us
    if s.frame_pairs > 0:
        s.mean_mse = mse_sum / s.frame_pairs
    if finite > 0:
        s.mean_psnr_db = db_sum / finite
        s.mean_psnr_linear = lin_sum / finite
    if s.frame_pairs > 0 and s.mean_mse > 0.0:
        s.psnr_db_of_mean_mse = 10.0 * math.log10(255.0 * 255.0 / s.mean_mse)
    if s.total_blocks_estimated > 0:
        s.avg_search_points = float(s.total_comparisons + s.total_dpd_steps) / float(s.total_blocks_estimated)
        if s.mean_psnr_linear and s.avg_search_points > 0.0:
            s.indicator = api.figure_of_merit(s.mean_psnr_linear, search_range, s.avg_search_points)
    return s


def dump_artifacts(index: int, pred: np.ndarray, resid: np.ndarray, dx: np.ndarray, dy: np.ndarray, directory: str):
    """pred_%04d.pgm, resid_%04d.pgm, vectors_%04d.txt (bench.cpp:77-93)."""
    os.makedirs(directory, exist_ok=True)
    seqio.write_gray_pgm(pred, os.path.join(directory, "pred_%04d.pgm" % index))
    seqio.write_gray_pgm(api.residual_to_gray(resid), os.path.join(directory, "resid_%04d.pgm" % index))
    rows, cols = dx.shape
    with open(os.path.join(directory, "vectors_%04d.txt" % index), "w") as f:
        for v in range(rows):
            for h in range(cols):
                f.write("%d %d %d %d\n" % (h, v, int(dx[v, h]), int(dy[v, h])))


def read_vectors_file(path: str, block_size: int) -> api.MotionField:  # bench.cpp:95-118
    entries = []
    with open(path) as f:
        toks = f.read().split()
    if len(toks) % 4:
        raise RuntimeError(f"malformed vector line in {path}")
    for i in range(0, len(toks), 4):
        h, v, dx, dy = (int(t) for t in toks[i:i + 4])
        if h < 0 or v < 0:
            raise RuntimeError(f"negative block coordinates in {path}")
        entries.append((h, v, dx, dy))
    if not entries:
        raise RuntimeError(f"empty vector file {path}")
    cols = max(e[0] for e in entries) + 1
    rows = max(e[1] for e in entries) + 1
    if len(entries) != cols * rows:
        raise RuntimeError(f"vector file does not cover the block grid: {path}")
    fld = api.MotionField(cols, rows, block_size)
    for h, v, dx, dy in entries:
        fld.set(h, v, (dx, dy))
    return fld


def run_experiment_arrays(cfg: ExperimentConfig, luma: np.ndarray, alpha: Optional[np.ndarray] = None,
                          device: int = 0) -> ExperimentResult:
    """run_experiment on in-memory frames ``[n, H, W]`` (masks likewise, 0/255)."""
    from . import batch

    n, H, W = luma.shape
    result = ExperimentResult()
    csv = open(cfg.csv_path, "w") if cfg.csv_path else None
    try:
        if csv:
            csv.write(CSV_HEADER + "\n")
        for algo in cfg.algos:
            scfg = algo_search_config(cfg, algo)
            bcfg = batch.BatchConfig(algo=algo, search=scfg, prs=cfg.prs, boundary_temporal=cfg.boundary_temporal)
            want_pred = bool(cfg.dump_dir)
            t = time.perf_counter()
            out = batch.run_sequences(bcfg, luma[None], None if alpha is None else alpha[None], want_pred=want_pred, device=device)
            dt_us = (time.perf_counter() - t) * 1e6
            recs, stats = out[0][0], out[1][0]
            pairs = n - scfg.ref_distance
            per = [int(dt_us // pairs)] * pairs
            reps = reports_from_stats(algo, stats, W * H, scfg.ref_distance, per)
            for i, r in enumerate(reps):
                if csv:
                    csv.write(csv_row(r) + "\n")
                if want_pred:
                    tau = r.frame
                    pred = out[2][0][i]
                    dump_artifacts(tau, pred, api.residual(luma[tau], pred), recs["dx"][i], recs["dy"][i],
                                   os.path.join(cfg.dump_dir, api.to_string(algo)))
            result.reports.extend(reps)
            result.summaries.append(summarize(algo, reps, scfg.search_range))
    finally:
        if csv:
            csv.close()
    return result


def run_experiment(cfg: ExperimentConfig, device: int = 0) -> ExperimentResult:  # bench.cpp:120-227
    cfg.validate()
    n = cfg.frames_used()
    W, H = cfg.source.width, cfg.source.height
    luma = seqio.stream_frames(cfg.source, n)  # straight into pinned memory
    alpha = None
    if cfg.masks.present():
        alpha = seqio.read_masks(cfg.masks, n, W, H, out=seqio.pinned_empty((n, H, W)))
    return run_experiment_arrays(cfg, luma, alpha, device)
