"""Parity against golden vectors made by the UNMODIFIED reference
(tests/golden/*.npz, from tools/make_golden.py running oracle/_ref).

The same fixtures pin the CPU oracle restatement (`port`, runs everywhere) and
check the CUDA path (`gpu`, -m gpu).  Integer results are compared bit-exact:
motion vectors, 4 x SAD, comparison / dpd / iteration counts, block classes,
per-pair SSE; prs_update doubles are compared exactly (same IEEE operations).
"""
import glob
import hashlib
import os

import numpy as np
import pytest

from backends import GpuBackend, PortBackend

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SEQ_FILES = sorted(glob.glob(os.path.join(GOLD, "seq_*.npz")))
# configs 3 and 5 at their real geometry and search range (S = 32 / 64):
# checked on the GPU only (tools/make_golden.py BIG_CASES)
BIG_FILES = sorted(glob.glob(os.path.join(GOLD, "big_*.npz")))
REC = np.dtype([("dx", "<i2"), ("dy", "<i2"), ("cost_q4", "<u4"), ("comparisons", "<u2"), ("dpd_steps", "<u2"), ("iterations", "u1"), ("type", "u1"), ("reserved", "<u2")])
STAT = np.dtype([(n, "<i8") for n in ("block_comparisons", "dpd_refinement_steps", "blocks_opaque", "blocks_boundary", "blocks_transparent", "sse")])


def backend(kind):
    return PortBackend() if kind == "port" else GpuBackend()


BACKENDS = [pytest.param("port"), pytest.param("gpu", marks=pytest.mark.gpu)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_seq(path):
    z = np.load(path)
    if "luma" in z:
        algo, S, bs, hp, d = (int(v) for v in z["config"])
        return z["luma"], z["alpha"], dict(algo=algo, S=S, bs=bs, halfpel=hp, ref_distance=d), z
    from paper_1002_1168_b200 import synth

    cid, seed, frames, algo, bs, S, hp = (int(v) for v in z["config"])
    luma, alpha = synth.config_sequence(cid, seed, None if frames < 0 else frames)
    assert sha(luma) == str(z["luma_sha"]) and sha(alpha) == str(z["alpha_sha"]), "config generator drifted"
    return luma, alpha, dict(algo=algo, S=S, bs=bs, halfpel=hp, ref_distance=2), z


@pytest.mark.parametrize("kind", BACKENDS)
@pytest.mark.parametrize("path", SEQ_FILES, ids=lambda p: os.path.basename(p)[4:-4])
def test_sequence_golden(kind, path):
    luma, alpha, c, z = load_seq(path)
    recs, stats = backend(kind).run_sequence(c["algo"], luma, alpha, c["bs"], c["S"], halfpel=c["halfpel"], ref_distance=c["ref_distance"])
    want_r = z["recs"].view(REC).reshape(recs.shape)
    want_s = z["stats"].view(STAT).reshape(stats.shape)
    bad = np.argwhere(recs != want_r)
    assert bad.size == 0, f"{len(bad)} record mismatches, first {tuple(bad[0])}: got {recs[tuple(bad[0])]} want {want_r[tuple(bad[0])]}"
    assert np.array_equal(stats, want_s)


@pytest.mark.gpu
@pytest.mark.parametrize("path", BIG_FILES, ids=lambda p: os.path.basename(p)[4:-4])
def test_big_golden_gpu(path):
    """1920x1088 (S = 32) and 3840x2160 (S = 64) sequences: the CUDA path's
    records and stats equal the reference's bit for bit (the S = 32 / 64
    es_kernel instantiations, the ring searches and PA at those ranges)."""
    luma, alpha, c, z = load_seq(path)
    recs, stats = backend("gpu").run_sequence(c["algo"], luma, alpha, c["bs"], c["S"])
    want_r = z["recs"].view(REC).reshape(recs.shape)
    want_s = z["stats"].view(STAT).reshape(stats.shape)
    bad = np.argwhere(recs != want_r)
    assert bad.size == 0, f"{len(bad)} record mismatches, first {tuple(bad[0])}: got {recs[tuple(bad[0])]} want {want_r[tuple(bad[0])]}"
    assert np.array_equal(stats, want_s)


@pytest.fixture(scope="module")
def blocks():
    return np.load(os.path.join(GOLD, "blocks.npz"))


@pytest.mark.parametrize("kind", BACKENDS)
def test_block_searches_golden(kind, blocks):
    be, P = backend(kind), blocks["planes"]
    for c, r, x0, y0, size, S, algo, mx, my, cmp, cost in blocks["block_search"]:
        mv, n = be.block_search(int(algo), P[c], P[r], int(x0), int(y0), int(size), int(S))
        assert (mv, n) == ((mx, my), cmp), (c, r, x0, y0, size, S, algo)


@pytest.mark.parametrize("kind", BACKENDS)
def test_brs_select_golden(kind, blocks):
    be, P, A = backend(kind), blocks["planes"], blocks["alphas"]
    for row in blocks["brs"]:
        c, r, x0, y0, size, btype, bt = (int(v) for v in row[:7])
        cands = [int(v) for v in row[7:15]]
        mv, kinds = be.brs_select(P[c], P[r], A[0], A[1], x0, y0, size, btype, cands, 7, bt)
        assert mv == (row[15], row[16]) and kinds == [int(v) for v in row[17:21]], row


@pytest.mark.parametrize("kind", BACKENDS)
def test_prs_refine_golden(kind, blocks):
    be, P = backend(kind), blocks["planes"]
    for row, log in zip(blocks["prs"], blocks["prs_logs"]):
        c, r, x0, y0, size, step, d0x, d0y, mx, my, dpd, n = (int(v) for v in row)
        mv, got_dpd, got_log = be.prs_refine(P[c], P[r], x0, y0, size, (d0x, d0y), 7, step=step)
        assert mv == (mx, my) and got_dpd == dpd and got_log == [int(v) for v in log[:n]], row


@pytest.mark.parametrize("kind", BACKENDS)
def test_sad_golden(kind, blocks):
    be, P, A = backend(kind), blocks["planes"], blocks["alphas"]
    for c, r, x0, y0, size, dx, dy, q4, shp in blocks["sad"]:
        assert be.sad_texture_q4(P[c], P[r], int(x0), int(y0), int(size), int(dx), int(dy)) == q4
        assert be.sad_shape(A[0], A[1], int(x0), int(y0), int(size), int(dx) & ~1, int(dy) & ~1) == shp


@pytest.mark.parametrize("kind", BACKENDS)
def test_predict_and_update_golden(kind, blocks):
    be, P = backend(kind), blocks["planes"]
    mv, ty, preds = blocks["pred_mv"], blocks["pred_types"], blocks["preds"]
    assert np.array_equal(be.predict(P[0], mv[0], ty[0], 8), preds[0])
    assert np.array_equal(be.predict(P[1], mv[1][:16], ty[1][:16], 16), preds[1])
    for c, r, x, y, dx, dy, ux, uy in blocks["prs_update"]:
        got = be.prs_update(P[int(c)], P[int(r)], int(x), int(y), (int(dx), int(dy)))
        assert got == (ux, uy)
