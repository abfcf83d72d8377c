"""The experiment driver (bench.cpp:120-227) and sequence I/O (video_io.cpp)
mirrored on the batched GPU path.

CPU: the host logic — CSV formatting, FrameReport/AlgoSummary arithmetic,
I420/Y4M/PGM readers — is pinned to the UNMODIFIED reference's own
run_experiment (oracle/_ref, built from /root/reference here): the reports
are rebuilt from the reference's per-pair stats with experiment.py and must
reproduce the reference's CSV (all columns but elapsed_us) and summaries
bit for bit.  GPU: the full run_experiment through the C ABI against the
committed golden CSV / summaries (tests/golden/experiment_*, made by
tools/make_golden.py from the reference).
"""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_1002_1168_b200 import api, experiment as ex, seqio, synth
from paper_1002_1168_b200._lib import stats_dtype

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ALGOS = [api.Algo.ES, api.Algo.TSS, api.Algo.FSS, api.Algo.DS, api.Algo.PA]


def write_case(tmp, cid=1, seed=11, frames=8, y4m=True):
    """A config-generator sequence as a Y4M (or I420) file plus P5 PGM masks."""
    luma, alpha = synth.config_sequence(cid, seed, frames)
    path = os.path.join(tmp, "seq.y4m" if y4m else "seq.yuv")
    seqio.write_i420(path, luma, y4m=y4m)
    for i in range(frames):
        # gray masks (0/200) exercise the binarisation threshold
        seqio.write_gray_pgm(np.where(alpha[i] > 0, 200, 0).astype(np.uint8), os.path.join(tmp, "mask%04d.pgm" % i))
    return path, os.path.join(tmp, "mask%04d.pgm"), luma, alpha


def cfg_for(S=7, halfpel=0):
    return api.SearchConfig(search_range=S, block_size=16, ref_distance=2, halfpel=bool(halfpel)), api.PrsConfig()


def test_fmt_double_matches_printf():
    libc = C.CDLL(None)
    buf = C.create_string_buffer(64)
    rng = np.random.default_rng(5)
    vals = list(rng.normal(0, 1e3, 200)) + list(rng.uniform(0, 60, 200)) + [0.0, 1.0, 48.130803608679102, 1e-300, 6.5e9, 1 / 3]
    for v in vals:
        libc.snprintf(buf, 64, b"%.17g", C.c_double(float(v)))
        assert ex.fmt_double(float(v)) == buf.value.decode()


def test_readers_roundtrip(tmp_path):
    path, pat, luma, alpha = write_case(str(tmp_path), frames=5)
    src = seqio.open_y4m(path)
    assert (src.width, src.height, src.frame_count) == (176, 144, 5)
    assert np.array_equal(seqio.read_frames(src), luma)
    assert np.array_equal(seqio.read_masks(seqio.MaskSource(pat), 5, 176, 144), np.where(alpha > 0, 255, 0))
    raw = os.path.join(str(tmp_path), "seq.yuv")
    seqio.write_i420(raw, luma)
    src2 = seqio.open_i420(raw, 176, 144)
    assert src2.frame_count == 5 and np.array_equal(seqio.read_frames(src2, 3), luma[:3])
    assert np.array_equal(seqio.stream_frames(src2, 4), luma[:4])
    assert np.array_equal(seqio.stream_frames(src), luma)
    with pytest.raises(ValueError):
        seqio.open_i420(raw, 100, 144)
    with pytest.raises(RuntimeError):
        seqio.parse_y4m_header("YUV4MPEG2 W176 H144 C444")
    with pytest.raises(RuntimeError):
        seqio.parse_y4m_header("YUV4MPEG2 W176")
    with open(raw, "ab") as f:
        f.write(b"x")
    with pytest.raises(RuntimeError):
        seqio.open_i420(raw, 176, 144)


def test_summary_of_infinite_psnr():
    # identical frames: every pair has SSE 0 -> psnr "inf", no finite mean
    r = ex.reports_from_stats(api.Algo.ES, np.zeros(3, stats_dtype()), 100, 2, [0, 0, 0])
    assert ex.csv_row(r[0]) == "2,ES,inf,0,nan,0,0,0,0,0"
    s = ex.summarize(api.Algo.ES, r, 7)
    assert s.mean_psnr_db is None and s.psnr_db_of_mean_mse is None and s.indicator is None


@pytest.mark.parametrize("y4m", [True, False])
def test_reports_reproduce_reference_run_experiment(tmp_path, refo, y4m):
    path, pat, luma, alpha = write_case(str(tmp_path), y4m=y4m)
    search, prs = cfg_for()
    csv_path = os.path.join(str(tmp_path), "ref.csv")
    c = oracle.make_cfg(algo=0, search_range=search.search_range, block_size=16, ref_distance=2)
    summ = refo.run_experiment(path, 1 if y4m else 0, 176, 144, pat, [int(a) for a in ALGOS], c, csv_path=csv_path)
    ref_rows = open(csv_path).read().splitlines()
    assert ref_rows[0] == ex.CSV_HEADER
    # our host logic over the reference's own per-pair stats
    src = seqio.open_sequence(path, 176, 144)
    frames = seqio.read_frames(src)
    masks = seqio.read_masks(seqio.MaskSource(pat), src.frame_count, 176, 144)
    cfg = ex.ExperimentConfig(source=src, masks=seqio.MaskSource(pat), algos=ALGOS, search=search, prs=prs)
    rows, k = [], 1
    for ai, algo in enumerate(ALGOS):
        s = ex.algo_search_config(cfg, algo)
        _, st = refo.run_sequence(oracle.make_cfg(algo=int(algo), search_range=s.search_range, block_size=s.block_size, ref_distance=2), frames, masks)
        elapsed = [int(r.split(",")[-1]) for r in ref_rows[k:k + len(st)]]
        k += len(st)
        reps = ex.reports_from_stats(algo, st, 176 * 144, 2, elapsed)
        rows += [ex.csv_row(r) for r in reps]
        sm = ex.summarize(algo, reps, s.search_range)
        got = [sm.frame_pairs, sm.mean_mse, sm.mean_psnr_db, sm.psnr_db_of_mean_mse, sm.mean_psnr_linear,
               sm.avg_search_points, sm.indicator, sm.total_comparisons, sm.total_dpd_steps, sm.total_blocks_estimated]
        for g, w in zip(got, summ[ai]):
            assert (g is None and math.isnan(w)) or g == w, (algo, got, summ[ai])
    assert rows == ref_rows[1:]


@pytest.mark.gpu
def test_gpu_run_experiment_matches_golden(tmp_path, me_gpu):
    gold_csv = open(os.path.join(GOLD, "experiment_cfg1.csv")).read().splitlines()
    gold_sum = json.load(open(os.path.join(GOLD, "experiment_cfg1.json")))
    path, pat, _, _ = write_case(str(tmp_path))
    search, prs = cfg_for()
    out_csv = os.path.join(str(tmp_path), "gpu.csv")
    dump = os.path.join(str(tmp_path), "dump")
    cfg = ex.ExperimentConfig(source=seqio.open_y4m(path), masks=seqio.MaskSource(pat), algos=ALGOS,
                              search=search, prs=prs, csv_path=out_csv, dump_dir=dump)
    res = ex.run_experiment(cfg)
    got = open(out_csv).read().splitlines()
    strip = lambda rows: [r.rsplit(",", 1)[0] for r in rows]
    assert strip(got) == strip(gold_csv)
    for sm, w in zip(res.summaries, gold_sum["summaries"]):
        g = [sm.frame_pairs, sm.mean_mse, sm.mean_psnr_db, sm.psnr_db_of_mean_mse, sm.mean_psnr_linear,
             sm.avg_search_points, sm.indicator, sm.total_comparisons, sm.total_dpd_steps, sm.total_blocks_estimated]
        assert [None if v is None else float(v) for v in g] == w
    # the dumped vector file parses back to the field
    fld = ex.read_vectors_file(os.path.join(dump, "PA", "vectors_0002.txt"), 8)
    assert (fld.cols, fld.rows) == (22, 18)
    assert os.path.getsize(os.path.join(dump, "ES", "pred_0002.pgm")) == len(b"P5\n176 144\n255\n") + 176 * 144
