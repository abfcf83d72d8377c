"""GPU parity tests: the CUDA path (through the C ABI) against the oracle
restatement on identical seeded inputs.  Integer results must be bit-exact
(MVs, per-block SAD x4, comparison / dpd / iteration counts, block classes,
SSE); the PSNR dB value is computed from the exact SSE on the host.
Run on a B200:  python -m pytest tests -m gpu
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ALGOS = [(4, 8), (4, 16), (0, 16), (1, 16), (2, 16), (3, 16)]


def noise(rng, h, w):
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)


def shift_clamped(base, sx, sy):
    h, w = base.shape
    ys = np.clip(np.arange(h) + sy, 0, h - 1)
    xs = np.clip(np.arange(w) + sx, 0, w - 1)
    return base[ys][:, xs]


def assert_recs(got, want, what=""):
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        i = tuple(bad[0])
        raise AssertionError(f"{what}: {len(bad)} record mismatches; first at {i}: got {got[i]} want {want[i]}")


@pytest.mark.parametrize("cfg_id", [1, 2])
@pytest.mark.parametrize("algo,bs", ALGOS)
def test_sequence_configs(me_gpu, port, cfg_id, algo, bs):
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config_sequence(cfg_id, 1000 + cfg_id)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=bs))
    recs, stats = me_gpu.run_sequences(cfg, luma[None], alpha[None])
    want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=16, block_size=bs), luma, alpha)
    assert_recs(recs[0], want_r, f"cfg{cfg_id} algo{algo} bs{bs}")
    assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("algo,bs", ALGOS)
def test_sequence_no_mask_and_pred(me_gpu, port, algo, bs):
    rng = np.random.default_rng(algo * 10 + bs)
    base = noise(rng, 96 + 32, 128 + 32)
    frames = np.stack([shift_clamped(base, 2 * t, -t)[16:16 + 96, 16:16 + 128] for t in range(5)])
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=7, block_size=bs, ref_distance=1))
    recs, stats, pred = me_gpu.run_sequences(cfg, frames[None], None, want_pred=True)
    want_r, want_s, want_p = port.run_sequence(oracle.make_cfg(algo=algo, search_range=7, block_size=bs, ref_distance=1), frames, None, want_pred=True)
    assert_recs(recs[0], want_r)
    assert np.array_equal(stats[0], want_s)
    assert np.array_equal(pred[0], want_p)


def test_batch_of_sequences_config4_small(me_gpu, port):
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config4_batch(6, 500, frames=8)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(6):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"seq {i}")
        assert np.array_equal(stats[i], want_s)


@pytest.mark.parametrize("contrast", ["full", "low"])
@pytest.mark.parametrize("bs", [8, 16])
def test_pa_tie_heavy_sequences(me_gpu, port, contrast, bs):
    """Low-contrast content makes PRS neighbour ties frequent, exercising the
    FP64 direction path (estimators.cpp:345-362)."""
    rng = np.random.default_rng(77 + bs)
    if contrast == "low":
        base = (100 + rng.integers(0, 3, size=(160, 192))).astype(np.uint8)
    else:
        base = noise(rng, 160, 192)
    frames = np.stack([shift_clamped(base, (t * 3) % 5 - 2, (t * 7) % 5 - 2)[16:144, 16:176] for t in range(8)])
    mask = np.zeros_like(frames)
    mask[:, 20:100, 30:120] = 255
    for halfpel in (0, 1):
        cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=8, block_size=bs, halfpel=bool(halfpel)))
        recs, stats = me_gpu.run_sequences(cfg, frames[None], mask[None])
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=8, block_size=bs, halfpel=halfpel), frames, mask)
        assert_recs(recs[0], want_r, f"halfpel={halfpel}")
        assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("algo", [0, 1, 2, 3])
@pytest.mark.parametrize("rng_s", [7, 16])
def test_block_search_random(me_gpu, port, algo, rng_s):
    rng = np.random.default_rng(2026 + algo)
    st = me_gpu.SearchStats()
    for trial in range(4):
        cur, ref = noise(rng, 64, 64), noise(rng, 64, 64)
        if trial == 1:  # smooth content: long descents, revisits
            cur = np.convolve(cur.ravel(), np.ones(9) / 9, "same").reshape(64, 64).astype(np.uint8)
            ref = shift_clamped(cur, 3, -2)
        for r in me_gpu.block_grid(64, 64, 16):
            st = me_gpu.SearchStats()
            fn = [me_gpu.full_search, me_gpu.tss_search, me_gpu.fss_search, me_gpu.ds_search][algo]
            mv = fn(cur, ref, r, me_gpu.SearchConfig(search_range=rng_s, block_size=16), st)
            want_mv, want_cmp, _ = port.block_search(algo, cur, ref, r.x0, r.y0, 16, rng_s)
            assert mv == tuple(want_mv) and st.block_comparisons == want_cmp, (trial, r)


def test_brs_select_random(me_gpu, port):
    rng = np.random.default_rng(11)
    for trial in range(40):
        cur, ref = noise(rng, 64, 64), noise(rng, 64, 64)
        ca = np.zeros((64, 64), np.uint8)
        ra = np.zeros((64, 64), np.uint8)
        ca[rng.integers(0, 30):rng.integers(34, 64), rng.integers(0, 30):rng.integers(34, 64)] = 255
        ra[rng.integers(0, 30):rng.integers(34, 64), rng.integers(0, 30):rng.integers(34, 64)] = 255
        size = 8 if trial % 2 else 16
        x0 = int(rng.integers(0, 64 // size)) * size
        y0 = int(rng.integers(0, 64 // size)) * size
        cands = [int(v) for v in rng.integers(-20, 21, size=8)]
        btype = int(rng.integers(1, 3))
        bt = int(trial % 3 == 0)
        cs = me_gpu.CandidateSet(tuple(cands[0:2]), tuple(cands[2:4]), tuple(cands[4:6]), tuple(cands[6:8]))
        log = []
        mv = me_gpu.brs_select(cur, ref, ca, ra, me_gpu.BlockRect(x0, y0, size), me_gpu.BlockType(btype), cs, me_gpu.SearchConfig(search_range=7, block_size=size), me_gpu.EstimateOptions(me_gpu.BoundaryTemporal(bt), log), me_gpu.SearchStats())
        want_mv, want_kinds = port.brs_select(cur, ref, ca, ra, x0, y0, size, btype, cands, 7, bt)
        assert mv == tuple(want_mv), trial
        assert [int(e.kind) for e in log] == want_kinds


@pytest.mark.parametrize("step", [2, 1])
@pytest.mark.parametrize("size", [8, 16])
def test_prs_refine_random(me_gpu, port, step, size):
    rng = np.random.default_rng(500 + step + size)
    for trial in range(30):
        if trial % 3 == 2:
            cur = (100 + rng.integers(0, 2, size=(64, 64))).astype(np.uint8)
            ref = (100 + rng.integers(0, 2, size=(64, 64))).astype(np.uint8)
        else:
            cur, ref = noise(rng, 64, 64), noise(rng, 64, 64)
        x0 = int(rng.integers(0, 64 // size)) * size
        y0 = int(rng.integers(0, 64 // size)) * size
        d0 = (int(rng.integers(-11, 12)), int(rng.integers(-11, 12)))
        st = me_gpu.SearchStats()
        log = []
        mv = me_gpu.prs_refine(cur, ref, me_gpu.BlockRect(x0, y0, size), d0, me_gpu.SearchConfig(search_range=7, block_size=size), me_gpu.PrsConfig(step=step), st, log)
        want_mv, want_dpd, want_log = port.prs_refine(cur, ref, x0, y0, size, d0, 7, step=step)
        assert mv == tuple(want_mv), trial
        assert st.dpd_refinement_steps == want_dpd
        assert [int(v * 4) for v in log] == want_log


def test_sad_texture_and_shape(me_gpu, port):
    rng = np.random.default_rng(3)
    cur, ref = noise(rng, 48, 64), noise(rng, 48, 64)
    ca = (noise(rng, 48, 64) > 128).astype(np.uint8) * 255
    ra = (noise(rng, 48, 64) > 100).astype(np.uint8) * 255
    for size in (8, 16):
        for x0, y0 in ((0, 0), (48 - size + 0, 16), (8, 32 - size + 16)):
            if x0 + size > 64 or y0 + size > 48:
                continue
            for dx in range(-21, 22, 3):
                for dy in (-19, -4, -1, 0, 1, 6, 25):
                    got = me_gpu.sad_texture(cur, ref, me_gpu.BlockRect(x0, y0, size), (dx, dy))
                    assert got == port.sad_texture(cur, ref, x0, y0, size, dx, dy)
                    if dx % 2 == 0 and dy % 2 == 0:
                        assert me_gpu.sad_shape(ca, ra, me_gpu.BlockRect(x0, y0, size), (dx, dy)) == port.sad_shape(ca, ra, x0, y0, size, dx, dy)
    with pytest.raises(ValueError):
        me_gpu.sad_shape(ca, ra, me_gpu.BlockRect(0, 0, 8), (1, 0))


def test_classify_binarize_predict_psnr(me_gpu, port):
    rng = np.random.default_rng(5)
    gray = noise(rng, 64, 96)
    assert np.array_equal(me_gpu.binarize(gray), port.binarize(gray))
    alpha = np.zeros((64, 96), np.uint8)
    alpha[10:50, 20:70] = 255
    for bs in (8, 16):
        assert np.array_equal(me_gpu.classify_blocks(alpha, bs), port.classify(alpha, bs))
    ref = noise(rng, 64, 96)
    cur = noise(rng, 64, 96)
    for bs in (8, 16):
        cols, rows = 96 // bs, 64 // bs
        mv = rng.integers(-40, 41, size=(cols * rows, 2)).astype(np.int32)
        types = rng.integers(0, 3, size=cols * rows).astype(np.uint8)
        f = me_gpu.MotionField(cols, rows, bs, vectors=mv, types=types)
        pred, sse = me_gpu.predict_frame(ref, f, me_gpu.SearchConfig(block_size=bs), cur=cur)
        want = port.predict_frame(ref, mv, types, bs)
        assert np.array_equal(pred, want)
        assert sse == int(((cur.astype(np.int64) - want) ** 2).sum())
    p = me_gpu.psnr(np.full((32, 32), 100, np.uint8), np.full((32, 32), 101, np.uint8))
    assert p.mse == 1.0 and abs(p.psnr_db - 48.1308) < 1e-3
    assert me_gpu.psnr(cur, cur).infinite()


def test_estimate_field_prev(me_gpu, port):
    rng = np.random.default_rng(9)
    base = noise(rng, 64, 64)
    cur, ref = shift_clamped(base, 2, 2), base
    prev = np.full((64, 2), 4, np.int32)
    pf = me_gpu.MotionField(8, 8, 8, vectors=prev.copy())
    f, st, recs = me_gpu.estimate_field(me_gpu.Algo.PA, cur, ref, None, None, pf, me_gpu.SearchConfig(block_size=8), me_gpu.PrsConfig(), return_records=True)
    want, wst = port.estimate_field(oracle.make_cfg(algo=4, search_range=7, block_size=8), cur, ref, prev_mv=prev)
    assert_recs(recs, want)
    assert f.at(0, 0) == (4, 4)
    flat = np.full((64, 64), 99, np.uint8)
    f2, _ = me_gpu.estimate_field(me_gpu.Algo.PA, flat, flat, None, None, pf, me_gpu.SearchConfig(block_size=8), me_gpu.PrsConfig())
    assert f2.at(0, 0) == (0, 0)


@pytest.mark.parametrize("levels", [(0, 255), (0, 100, 255)])
def test_host_path_mask_packing(me_gpu, port, levels):
    """The host-pointer path ships binary masks bit-packed (expanded on the
    device); a mask with other values must go as bytes — both bit-exact."""
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config4_batch(9, 900, frames=5)
    if len(levels) == 3:  # make some object pixels a different nonzero value
        alpha = alpha.copy()
        alpha[:, :, ::3, ::5] = np.where(alpha[:, :, ::3, ::5] > 0, 100, 0)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in (0, 4, 8):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"seq {i}")
        assert np.array_equal(stats[i], want_s)


@pytest.mark.parametrize("odd", [False, True])
def test_estimate_field_random_prev(me_gpu, port, odd):
    """External prev fields: integer-pel ones take the fast PA kernels, a
    half-pel one the generic kernel; both bit-exact."""
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config_sequence(1, 77, 4)
    rng = np.random.default_rng(3 + odd)
    prev = rng.integers(-12, 13, size=(22 * 18, 2)).astype(np.int32)
    prev = prev | 1 if odd else prev & ~1
    pf = me_gpu.MotionField(22, 18, 8, vectors=prev.copy())
    f, st, recs = me_gpu.estimate_field(me_gpu.Algo.PA, luma[2], luma[0], alpha[2], alpha[0], pf,
                                        me_gpu.SearchConfig(search_range=16, block_size=8), me_gpu.PrsConfig(), return_records=True)
    want, wst = port.estimate_field(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[2], luma[0], alpha[2], alpha[0], prev_mv=prev)
    assert_recs(recs, want)


@pytest.fixture
def tuning(me_gpu):
    """Sets this thread's context tuning for one test (me_b200_ctx_set_tuning), restored after."""
    from paper_1002_1168_b200 import _lib

    saved = []

    def set_(**kw):
        saved.append(_lib.set_tuning(0, **kw))

    yield set_
    if saved:
        _lib.restore_tuning(saved[0], 0)


@pytest.mark.parametrize("key", [1, 0, -1])
@pytest.mark.parametrize("mode", ["auto", "fast", "hybrid", "hybrid-static"])
def test_pa_list_keys(me_gpu, port, mode, key, tuning):
    """The PA list ordered by the plain wavefront step t = h + 2v + p
    (pa_key_plain 1) or by t - tmin(sequence) (0: batches up to 60 000 blocks
    per step, -1: any width): the same records and stats.  The batch mixes
    sequences whose first estimated block comes at different steps, one
    sequence without masks (every block opaque: tmin 0) and one whose masks are
    empty (no estimated block: no tmin)."""
    from paper_1002_1168_b200 import synth

    tuning(pa_schedule=mode.split("-static")[0], pa_wide_blocks=4, pa_static_claim=int(mode.endswith("-static")), pa_key_plain=key)
    luma, alpha = synth.config4_batch(7, 910, frames=8)
    alpha[5] = 255
    alpha[6] = 0
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(7):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"{mode} key {key} seq {i}")
        assert np.array_equal(stats[i], want_s)


@pytest.mark.parametrize("S", [12, 24, 32, 48])
@pytest.mark.parametrize("bs", [8, 16])
def test_es_blocks_per_pass(me_gpu, port, S, bs):
    """es_kernel's small-window path (NB = 4 / 2 blocks per CTA pass, the
    compile-time and generic row strides) and its banded large-window path,
    on a batch whose block count is not a multiple of NB."""
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config4_batch(3, 5200 + S + bs, frames=4)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.ES, search=me_gpu.SearchConfig(search_range=S, block_size=bs))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(3):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=int(me_gpu.Algo.ES), search_range=S, block_size=bs), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"ES S{S} bs{bs} seq {i}")
        assert np.array_equal(stats[i], want_s)


@pytest.mark.parametrize("ctas", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("window", [0, 1])
def test_pa_fast_ctas_per_sm(me_gpu, port, ctas, window, tuning):
    """pa_fast_kernel at every CTAs-per-SM instantiation the schedule picks by
    batch width (1 for single sequences, 2 / 3 / 4 for wider batches and the
    hybrid's head and tail; 5 / 6 by tuning), with the staged window and with
    per-candidate patches."""
    from paper_1002_1168_b200 import synth

    tuning(pa_schedule="fast", pa_fast_ctas=ctas, pa_fast_patches=1 - window)
    luma, alpha = synth.config4_batch(3, 4100 + ctas, frames=5)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(3):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"ctas {ctas} window {window} seq {i}")
        assert np.array_equal(stats[i], want_s)


@pytest.mark.parametrize("bt,it", [(0, 4), (1, 4), (0, 7)])
@pytest.mark.parametrize("mode", ["fast", "duo", "duo-hybrid", "hybrid", "warp", "hybrid-static"])
def test_pa_kernel_modes(me_gpu, port, mode, bt, it, tuning):
    """Every PA kernel schedule (one block per warp, two per warp, the hybrid
    splits of the sorted list with two or four blocks per warp in the wide
    range, the generic kernel) on the same batch; the hybrids' wide threshold
    is lowered so all three of their ranges are used.  Also with
    BoundaryTemporal::Shape and a longer PRS iteration limit."""
    from paper_1002_1168_b200 import synth

    tuning(pa_schedule=mode.split("-static")[0], pa_wide_blocks=4, pa_static_claim=int(mode.endswith("-static")))
    luma, alpha = synth.config4_batch(5, 700, frames=6)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8),
                             prs=me_gpu.PrsConfig(max_iterations=it), boundary_temporal=me_gpu.BoundaryTemporal(bt))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(5):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8, boundary_temporal=bt, max_iterations=it), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"{mode} bt{bt} it{it} seq {i}")
        assert np.array_equal(stats[i], want_s)


def test_concurrent_host_threads(me_gpu, port):
    """Each host thread gets its own context (stream + buffers): concurrent
    calls on distinct data stay correct, as the reference's API promises."""
    import threading

    from paper_1002_1168_b200 import synth

    jobs = [(algo, bs, seed) for seed in (41, 42) for algo, bs in ((4, 8), (0, 16), (2, 16))]
    out, errs = {}, []

    def work(algo, bs, seed):
        try:
            luma, alpha = synth.config_sequence(1, seed, 6)
            cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=bs))
            out[(algo, bs, seed)] = (luma, alpha, me_gpu.run_sequences(cfg, luma[None], alpha[None]))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    threads = [threading.Thread(target=work, args=j) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for (algo, bs, seed), (luma, alpha, (recs, stats)) in out.items():
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=16, block_size=bs), luma, alpha)
        assert_recs(recs[0], want_r, f"algo{algo} seed{seed}")
        assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("mode", ["fast", "fast-patches", "duo", "duo-hybrid", "hybrid"])
@pytest.mark.parametrize("shape", [(16, 16), (48, 32), (64, 80)])
def test_pa_kernel_modes_small_frames(me_gpu, port, mode, shape, tuning):
    """Every PA schedule on frames a few blocks wide (patches clipped by every
    frame edge, windows smaller than the search range), with masks mixing
    transparent, opaque and boundary blocks and strong motion; `fast-patches`
    is pa_fast_kernel with per-candidate patches instead of the staged window."""
    H, W = shape
    patches = mode == "fast-patches"
    tuning(pa_schedule="fast" if patches else mode, pa_wide_blocks=1, pa_no_smem_pair=1, pa_fast_patches=int(patches))
    rng = np.random.default_rng(H * 1000 + W)
    n_seq, F = 6, 5
    base = noise(rng, H + 40, W + 40)
    luma = np.stack([np.stack([shift_clamped(base, int(rng.integers(-6, 7)), int(rng.integers(-6, 7)))[20:20 + H, 20:20 + W]
                               for _ in range(F)]) for _ in range(n_seq)])
    alpha = np.zeros_like(luma)
    alpha[0] = 255  # all opaque
    alpha[2, :, H // 4: 3 * H // 4, W // 3:] = 255  # boundary blocks
    alpha[3] = (rng.integers(0, 4, size=alpha[3].shape) == 0) * 255  # speckle: mostly boundary
    alpha[4, :, :, : W // 2] = 255
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha.astype(np.uint8))
    for i in range(n_seq):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i].astype(np.uint8))
        assert_recs(recs[i], want_r, f"{mode} {shape} seq {i}")
        assert np.array_equal(stats[i], want_s)


def test_batch_beyond_4gib(me_gpu, port):
    """A batch whose frames span more than 4 GiB of device memory (the PA
    kernels use 32-bit plane offsets; the library runs it as consecutive
    sub-batches below 4 GiB): the last sequences, whose pixels lie past
    4 GiB, match the oracle, and so does the first."""
    import torch

    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth

    free, _ = torch.cuda.mem_get_info()
    n_seq, F = 1440, 30  # 1440 x 30 x 352 x 288 = 4.38 GB of luma (and as much alpha)
    if free < 14 * 2**30:
        pytest.skip("needs ~14 GB of free device memory")
    luma, alpha = synth.config4_batch_dev(n_seq, 4100, frames=F)
    assert luma.numel() > 2**32
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    recs, stats = B.run_sequences_dev(cfg, luma, alpha)
    torch.cuda.synchronize()
    for i in (0, n_seq - 2, n_seq - 1):
        got_r = recs[i].cpu().numpy().view(_lib_rec_dtype()).reshape(recs.shape[1:4])
        got_s = stats[i].cpu().numpy().view(_lib_stats_dtype()).reshape(-1)
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i].cpu().numpy(), alpha[i].cpu().numpy())
        assert_recs(got_r, want_r, f"seq {i}")
        assert np.array_equal(got_s, want_s)
    del luma, alpha, recs, stats
    torch.cuda.empty_cache()


def _lib_rec_dtype():
    from paper_1002_1168_b200 import _lib

    return _lib.rec_dtype()


def _lib_stats_dtype():
    from paper_1002_1168_b200 import _lib

    return _lib.stats_dtype()


@pytest.mark.parametrize("algo", [1, 2, 3])
@pytest.mark.parametrize("bs", [8, 16])
@pytest.mark.parametrize("shape", [(96, 144), (64, 96)])
def test_ring_searches_batched(me_gpu, port, algo, bs, shape):
    """TSS / FSS / DS through the batched ring kernel at both block sizes
    (every displaced reference row is unaligned for odd vectors: the kernel's
    aligned-load path), an odd number of 16-pixel columns, and a smooth moving
    texture (long descents, revisited positions)."""
    h, w = shape
    rng = np.random.default_rng(algo * 100 + bs + h)
    base = noise(rng, h + 40, w + 40)
    base = np.convolve(base.ravel(), np.ones(5) / 5, "same").reshape(base.shape).astype(np.uint8)
    frames = np.stack([shift_clamped(base, 3 * t, -2 * t)[20:20 + h, 20:20 + w] for t in range(5)])
    for rng_s in (7, 16):
        cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=rng_s, block_size=bs, ref_distance=1))
        recs, stats = me_gpu.run_sequences(cfg, frames[None], None)
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=rng_s, block_size=bs, ref_distance=1), frames, None)
        assert_recs(recs[0], want_r, f"algo{algo} bs{bs} {shape} S{rng_s}")
        assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("algo", [1, 2, 3])
@pytest.mark.parametrize("bs", [8, 16])
@pytest.mark.parametrize("rng_s", [1, 2, 5, 9, 33])
def test_ring_staged_region_ranges(me_gpu, port, algo, bs, rng_s):
    """The ring kernel's persistent staged region (8 pels around a centre,
    restaged when a ring leaves it) against windows smaller and larger than
    it, clipped at every frame edge (QCIF-sized frame, every block estimated),
    with fast motion so DS walks far and TSS's big rings leave the region."""
    rng = np.random.default_rng(7 * algo + bs + 100 * rng_s)
    h, w = 80, 112
    base = noise(rng, h + 80, w + 80)
    base = np.convolve(base.ravel(), np.ones(3) / 3, "same").reshape(base.shape).astype(np.uint8)
    frames = np.stack([shift_clamped(base, 7 * t, -5 * t)[40:40 + h, 40:40 + w] for t in range(4)])
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=rng_s, block_size=bs, ref_distance=1))
    recs, stats = me_gpu.run_sequences(cfg, frames[None], None)
    want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=rng_s, block_size=bs, ref_distance=1), frames, None)
    assert_recs(recs[0], want_r, f"algo{algo} bs{bs} S{rng_s}")
    assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("algo", [1, 2, 3])
@pytest.mark.parametrize("bs", [8, 16])
def test_ring_single_block_odd_width(me_gpu, port, algo, bs):
    """The per-block entry points on a frame whose width is not a multiple of
    4 (no row of either plane is word-aligned)."""
    rng = np.random.default_rng(31 * algo + bs)
    base = noise(rng, 90, 110)
    base = np.convolve(base.ravel(), np.ones(7) / 7, "same").reshape(base.shape).astype(np.uint8)
    cur, ref = base[10:60, 10:80].copy(), base[13:63, 8:78].copy()  # 50 x 70
    fn = [None, me_gpu.tss_search, me_gpu.fss_search, me_gpu.ds_search][algo]
    rects = [me_gpu.BlockRect(x0, y0, bs, x0 // bs, y0 // bs) for y0 in range(0, 50 - bs + 1, bs) for x0 in range(0, 70 - bs + 1, bs)]
    for r in rects:
        for rng_s in (7, 16):
            st = me_gpu.SearchStats()
            mv = fn(cur, ref, r, me_gpu.SearchConfig(search_range=rng_s, block_size=bs), st)
            want_mv, want_cmp, _ = port.block_search(algo, cur, ref, r.x0, r.y0, bs, rng_s)
            assert mv == tuple(want_mv) and st.block_comparisons == want_cmp, (r, rng_s)


PA_VARIANTS = [
    # (bs, halfpel, boundary_temporal, max_iter, step, eps, theta)
    (8, 0, 1, 4, 2, 0.5, 2.0),    # BoundaryTemporal::Shape: T scored by sad_shape on boundary blocks
    (16, 0, 1, 4, 2, 0.5, 2.0),
    (8, 1, 1, 4, 1, 0.5, 2.0),    # half-pel + Shape
    (16, 1, 0, 4, 1, 0.5, 2.0),
    (8, 0, 0, 1, 2, 0.5, 2.0),    # one PRS iteration
    (8, 0, 0, 9, 2, 0.5, 2.0),    # long descents (more centres than the register-tracked three)
    (16, 1, 0, 6, 1, 0.25, 1.0),  # other epsilon / theta: the FP64 probing direction changes tie breaks
    (8, 0, 0, 4, 2, 1.0, 0.5),
]


@pytest.mark.parametrize("bs,hp,bt,it,step,eps,theta", PA_VARIANTS)
def test_pa_config_variants(me_gpu, port, bs, hp, bt, it, step, eps, theta):
    """The PA variants the API exposes but the benchmark configs do not
    exercise: BoundaryTemporal::Shape, half-pel mode,
    PRS iteration limits, epsilon and theta — bit-exact records and stats on
    config 1 and config 2 sequences (every kernel schedule the variant takes)."""
    from paper_1002_1168_b200 import synth

    for cfg_id, seed in ((1, 4100 + bs), (2, 4200 + bs)):
        luma, alpha = synth.config_sequence(cfg_id, seed, 6)
        cfg = me_gpu.BatchConfig(
            algo=me_gpu.Algo.PA,
            search=me_gpu.SearchConfig(search_range=16, block_size=bs, halfpel=bool(hp)),
            prs=me_gpu.PrsConfig(epsilon=eps, theta=theta, max_iterations=it, step=step),
            boundary_temporal=me_gpu.BoundaryTemporal(bt),
        )
        recs, stats = me_gpu.run_sequences(cfg, luma[None], alpha[None])
        want_r, want_s = port.run_sequence(
            oracle.make_cfg(algo=4, search_range=16, block_size=bs, halfpel=hp, boundary_temporal=bt,
                            max_iterations=it, step=step, epsilon=eps, theta=theta), luma, alpha)
        assert_recs(recs[0], want_r, f"cfg{cfg_id} bs{bs} hp{hp} bt{bt} it{it} step{step} eps{eps} theta{theta}")
        assert np.array_equal(stats[0], want_s)


@pytest.mark.parametrize("key", [1, -1])
@pytest.mark.parametrize("bs,hp,bt,it,step,eps,theta", PA_VARIANTS[:4])
def test_pa_config_variants_batched(me_gpu, port, bs, hp, bt, it, step, eps, theta, key, tuning):
    """The same variants on a batch of config-4 sequences (the generic and
    fast kernels over a multi-sequence list, with the plain and the aligned
    list keys)."""
    from paper_1002_1168_b200 import synth

    tuning(pa_key_plain=key)
    luma, alpha = synth.config4_batch(4, 4300 + bs + hp, frames=5)
    cfg = me_gpu.BatchConfig(
        algo=me_gpu.Algo.PA,
        search=me_gpu.SearchConfig(search_range=16, block_size=bs, halfpel=bool(hp)),
        prs=me_gpu.PrsConfig(epsilon=eps, theta=theta, max_iterations=it, step=step),
        boundary_temporal=me_gpu.BoundaryTemporal(bt),
    )
    recs, stats = me_gpu.run_sequences(cfg, luma, alpha)
    for i in range(4):
        want_r, want_s = port.run_sequence(
            oracle.make_cfg(algo=4, search_range=16, block_size=bs, halfpel=hp, boundary_temporal=bt,
                            max_iterations=it, step=step, epsilon=eps, theta=theta), luma[i], alpha[i])
        assert_recs(recs[i], want_r, f"seq {i} bs{bs} hp{hp} bt{bt} it{it} key{key}")
        assert np.array_equal(stats[i], want_s)


# ---------------------------------------------------------------------------
# Sharding entry points and concurrency


@pytest.mark.parametrize("algo", [0, 1, 2, 3])
def test_row_bands_sum_to_the_whole(me_gpu, port, algo):
    """me_b200_run_band_dev: the row bands of a batch reproduce the whole
    batch's records, and their stats (SearchStats + SSE) add up to it."""
    import torch

    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config_sequence(2, 61, 6)
    lt = torch.from_numpy(luma[None].copy()).cuda()
    at = torch.from_numpy(alpha[None].copy()).cuda()
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=16))
    full_r, full_s = B.run_sequences_dev(cfg, lt, at)
    pairs, rows = 4, luma.shape[1] // 16
    recs = torch.zeros_like(full_r)
    total = torch.zeros((1, pairs, 6), dtype=torch.int64, device="cuda")
    for r0, r1 in ((0, 5), (5, 6), (6, rows)):
        st = torch.empty((1, pairs, 48), dtype=torch.uint8, device="cuda")
        B.run_band_dev(cfg, lt, at, r0, r1, recs, st)
        total += st.view(torch.int64).view(1, pairs, 6)
    torch.cuda.synchronize()
    assert torch.equal(recs, full_r)
    assert torch.equal(total, full_s.view(torch.int64).view(1, pairs, 6))
    want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=16, block_size=16), luma, alpha)
    assert_recs(recs[0].cpu().numpy().view(_lib_rec_dtype()).reshape(want_r.shape), want_r)


def test_row_band_rejects_pa_and_bad_bands(me_gpu):
    import torch

    from paper_1002_1168_b200 import batch as B

    lt = torch.zeros((1, 4, 64, 64), dtype=torch.uint8, device="cuda")
    recs = torch.zeros((1, 2, 8, 8, 16), dtype=torch.uint8, device="cuda")
    st = torch.zeros((1, 2, 48), dtype=torch.uint8, device="cuda")
    pa = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=8, block_size=8))
    with pytest.raises(ValueError):
        B.run_band_dev(pa, lt, None, 0, 4, recs, st)
    es = me_gpu.BatchConfig(algo=me_gpu.Algo.ES, search=me_gpu.SearchConfig(search_range=8, block_size=8))
    for r0, r1 in ((0, 0), (-1, 3), (2, 9)):
        with pytest.raises(ValueError):
            B.run_band_dev(es, lt, None, r0, r1, recs, st)


@pytest.mark.parametrize("algo,bs", [(4, 8), (0, 16), (3, 16)])
def test_multi_device_entry(me_gpu, port, algo, bs):
    """me_b200_run_sequences_multi over the visible devices equals the
    single-device call (a lone baseline sequence shards by frame pairs)."""
    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth

    n = me_gpu.device_count()
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=bs))
    luma, alpha = synth.config4_batch(3, 700, 6) if algo == 4 else [x[None] for x in synth.config_sequence(2, 71, 6)]
    want = me_gpu.run_sequences(cfg, luma, alpha)
    got = B.run_sequences_multi(cfg, luma, alpha, n_gpus=n)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    with pytest.raises(ValueError):
        B.run_sequences_multi(cfg, luma, alpha, n_gpus=n + 1)


def test_concurrent_large_batches(me_gpu, port):
    """Two host threads each run a 64-sequence config-4 batch on one GPU at
    the same time.  Both select the persistent PA grids (hybrid head / quad
    middle / tail); with in-order claiming neither depends on its grid being
    fully resident, so the two grids sharing the device both finish, with
    results equal to the oracle's."""
    import threading

    from paper_1002_1168_b200 import synth

    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    inputs = [synth.config4_batch(64, 1000 + 100 * k, 8) for k in range(2)]
    out, errs = [None, None], []

    def work(k):
        try:
            for _ in range(3):
                out[k] = me_gpu.run_sequences(cfg, *inputs[k])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=120)
        assert not t.is_alive(), "concurrent batches did not finish"
    assert not errs, errs
    c = oracle.make_cfg(algo=4, search_range=16, block_size=8)
    for k in range(2):
        luma, alpha = inputs[k]
        for i in (0, 31, 63):
            want_r, want_s = port.run_sequence(c, luma[i], alpha[i])
            assert_recs(out[k][0][i], want_r, f"batch {k} seq {i}")
            assert np.array_equal(out[k][1][i], want_s)


# ---------------------------------------------------------------------------
# Bit-packed binary masks (north star: BAB shape matching with popc(XOR))


@pytest.mark.parametrize("mode", ["auto", "fast", "hybrid", "warp", "duo"])
def test_pa_bit_packed_masks(me_gpu, port, mode, tuning):
    """PA with the masks as device bit planes equals the byte-mask path and
    the oracle, under every schedule (fast / quad read the bits; the others
    get them expanded)."""
    import torch

    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth

    tuning(pa_schedule=mode, pa_wide_blocks=4)
    luma, alpha = synth.config4_batch(4, 810, frames=6)
    lt, at = torch.from_numpy(luma).cuda(), torch.from_numpy(alpha).cuda()
    bits, binary = B.pack_mask_dev(at)
    assert binary
    assert np.array_equal(bits.cpu().numpy(), np.packbits(alpha != 0, axis=-1, bitorder="little"))
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.PA, search=me_gpu.SearchConfig(search_range=16, block_size=8))
    r_bits, s_bits = B.run_sequences_bits_dev(cfg, lt, bits)
    r_byte, s_byte = B.run_sequences_dev(cfg, lt, at)
    torch.cuda.synchronize()
    assert torch.equal(r_bits, r_byte) and torch.equal(s_bits, s_byte)
    got = r_bits.cpu().numpy().view(_lib_rec_dtype()).reshape(r_bits.shape[:4])
    for i in (0, 3):
        want_r, want_s = port.run_sequence(oracle.make_cfg(algo=4, search_range=16, block_size=8), luma[i], alpha[i])
        assert_recs(got[i], want_r, f"{mode} seq {i}")


@pytest.mark.parametrize("algo,bs", [(0, 16), (1, 16), (3, 8), (4, 16)])
def test_bit_packed_masks_other_algos(me_gpu, port, algo, bs):
    import torch

    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth

    luma, alpha = synth.config_sequence(2, 83, 5)
    lt, at = torch.from_numpy(luma[None].copy()).cuda(), torch.from_numpy(alpha[None].copy()).cuda()
    bits, binary = B.pack_mask_dev(at)
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=bs))
    r, s = B.run_sequences_bits_dev(cfg, lt, bits)
    want_r, want_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=16, block_size=bs), luma, alpha)
    assert_recs(r[0].cpu().numpy().view(_lib_rec_dtype()).reshape(want_r.shape), want_r)
    assert np.array_equal(s[0].cpu().numpy().view(_lib_stats_dtype()).reshape(-1), want_s)


def test_pack_mask_dev_detects_non_binary(me_gpu):
    import torch

    from paper_1002_1168_b200 import batch as B

    a = torch.zeros((2, 64, 64), dtype=torch.uint8, device="cuda")
    a[0, 10:20, 5:40] = 255
    assert B.pack_mask_dev(a)[1]
    a[1, 3, 3] = 100
    bits, binary = B.pack_mask_dev(a)
    assert not binary
    assert np.array_equal(bits.cpu().numpy(), np.packbits(a.cpu().numpy() != 0, axis=-1, bitorder="little"))


# ---------------------------------------------------------------------------
# Large search ranges (the ES tie-break key and the 16-bit record
# count at S >= 128) and the S <= 255 implementation limit


@pytest.mark.parametrize("S", [127, 128, 200, 255])
@pytest.mark.parametrize("algo", [0, 3])
def test_large_search_range(me_gpu, port, S, algo):
    """ES / DS at S >= 128 on a 544 x 528 frame: MVs and the exact comparison
    count (ES window area up to 511^2 > 65535) match the oracle.  Smooth,
    tie-prone content so the Manhattan tie-break (|dx| + |dy| up to 2S, 9
    bits of the key) decides."""
    rng = np.random.default_rng(S + algo)
    base = np.convolve(noise(rng, 528, 560).ravel(), np.ones(15) / 15, "same").reshape(528, 560)
    cur = (base[:, :544] // 16 * 16).astype(np.uint8)
    ref = np.ascontiguousarray(shift_clamped(cur, 9, -5))
    cur = np.ascontiguousarray(cur)
    for x0, y0 in ((0, 0), (256, 256), (528, 512), (272, 16)):
        st = me_gpu.SearchStats()
        fn = me_gpu.full_search if algo == 0 else me_gpu.ds_search
        mv = fn(cur, ref, me_gpu.BlockRect(x0, y0, 16), me_gpu.SearchConfig(search_range=S, block_size=16), st)
        want_mv, want_cmp, _ = port.block_search(algo, cur, ref, x0, y0, 16, S)
        assert mv == tuple(want_mv) and st.block_comparisons == want_cmp, (S, x0, y0)


def test_search_range_limit(me_gpu):
    rng = np.random.default_rng(3)
    cur = noise(rng, 64, 64)
    with pytest.raises(ValueError):
        me_gpu.full_search(cur, cur, me_gpu.BlockRect(0, 0, 16), me_gpu.SearchConfig(search_range=256, block_size=16), me_gpu.SearchStats())


def test_es_batch_large_range_records(me_gpu, port):
    """The batched ES path at S = 160: records (comparisons saturate at
    65535 in the 16-bit field) and the exact int64 per-pair stats."""
    import torch

    from paper_1002_1168_b200 import batch as B

    rng = np.random.default_rng(160)
    base = np.convolve(noise(rng, 352, 352).ravel(), np.ones(7) / 7, "same").reshape(352, 352).astype(np.uint8)
    luma = np.stack([base, shift_clamped(base, 2, 1), shift_clamped(base, 40, -33)])
    alpha = np.zeros_like(luma)
    alpha[:, 96:224, 64:288] = 255
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo.ES, search=me_gpu.SearchConfig(search_range=160, block_size=16, ref_distance=2))
    r, s = B.run_sequences_dev(cfg, torch.from_numpy(luma[None].copy()).cuda(), torch.from_numpy(alpha[None].copy()).cuda())
    got_r = r[0].cpu().numpy().view(_lib_rec_dtype()).reshape(1, 22, 22)
    got_s = s[0].cpu().numpy().view(_lib_stats_dtype()).reshape(-1)
    want_r, want_s = port.run_sequence(oracle.make_cfg(algo=0, search_range=160, block_size=16), luma, alpha)
    assert np.array_equal(got_s, want_s)
    for f in ("dx", "dy", "cost_q4", "type"):
        assert np.array_equal(got_r[f], want_r[f]), f
    assert np.array_equal(got_r["comparisons"], want_r["comparisons"])  # both saturate at 65535
    assert got_r["comparisons"].max() == 65535


# ---------------------------------------------------------------------------
# Streaming I/O: a sequence file through the GPU in chunks


@pytest.mark.parametrize("algo,bs,chunk", [(4, 8, 5), (4, 8, 7), (0, 16, 6), (3, 16, 4)])
def test_estimate_stream_equals_whole_sequence(me_gpu, port, tmp_path, algo, bs, chunk):
    """seqio.estimate_stream (pinned slots filled by a reader thread, H2D on a
    copy stream, chunks chained through the temporal candidate) gives exactly
    the whole-sequence result, and the oracle's."""
    from paper_1002_1168_b200 import seqio, synth

    luma, alpha = synth.config_sequence(2, 95, 17)
    path = str(tmp_path / "seq.yuv")
    seqio.write_i420(path, luma)
    for i in range(luma.shape[0]):
        seqio.write_gray_pgm(alpha[i], str(tmp_path / f"mask_{i:03d}.pgm"))
    src = seqio.open_sequence(path, luma.shape[2], luma.shape[1])
    masks = seqio.MaskSource(pattern=str(tmp_path / "mask_%03d.pgm"))
    cfg = me_gpu.BatchConfig(algo=me_gpu.Algo(algo), search=me_gpu.SearchConfig(search_range=16, block_size=bs))
    r, s = seqio.estimate_stream(src, cfg, masks, chunk=chunk)
    want_r, want_s = me_gpu.run_sequences(cfg, luma[None], alpha[None])
    assert np.array_equal(r, want_r[0]) and np.array_equal(s, want_s[0])
    o_r, o_s = port.run_sequence(oracle.make_cfg(algo=algo, search_range=16, block_size=bs), luma, alpha)
    assert_recs(r, o_r, "stream")


# ---------------------------------------------------------------------------
# Seeded fuzz: random geometry, configuration and content against the oracle


def _fuzz_case(seed):
    rng = np.random.default_rng(seed)
    W, H = 16 * int(rng.integers(2, 9)), 16 * int(rng.integers(2, 8))
    F = int(rng.integers(3, 7))
    d = int(rng.integers(1, min(3, F - 1) + 1))
    algo = int(rng.integers(0, 5))
    bs = int(rng.choice([8, 16]))
    S = int(rng.integers(1, 25))
    hp = int(algo == 4 and rng.random() < 0.3)
    bt = int(algo == 4 and rng.random() < 0.3)
    it = int(rng.integers(1, 8))
    step = 1 if hp else int(rng.choice([1, 2, 2]))
    eps = float(rng.choice([0.25, 0.5, 1.0]))
    theta = float(rng.choice([0.5, 2.0, 4.0]))
    base = np.convolve(noise(rng, H + 32, W + 32).ravel(), np.ones(int(rng.integers(1, 12))) / 1.0, "same")
    base = (base.reshape(H + 32, W + 32) // int(rng.integers(1, 64))).astype(np.uint8)
    sh = rng.integers(-6, 7, size=(F, 2))
    luma = np.stack([base[16 + sh[t, 1]:16 + sh[t, 1] + H, 16 + sh[t, 0]:16 + sh[t, 0] + W] for t in range(F)])
    kind = int(rng.integers(0, 3))  # no mask, binary mask, non-binary mask
    alpha = None
    if kind:
        alpha = np.zeros_like(luma)
        for t in range(F):
            x0, y0 = int(rng.integers(0, W // 2)), int(rng.integers(0, H // 2))
            alpha[t, y0:y0 + int(rng.integers(4, H)), x0:x0 + int(rng.integers(4, W))] = 255
            if kind == 2:
                alpha[t, rng.integers(0, H, 5), rng.integers(0, W, 5)] = rng.integers(1, 255, 5).astype(np.uint8)
    return dict(luma=np.ascontiguousarray(luma), alpha=alpha, algo=algo, bs=bs, S=S, halfpel=hp, ref_distance=d, bt=bt,
                max_iter=it, step=step, eps=eps, theta=theta)


@pytest.mark.parametrize("seed", range(200))
def test_fuzz_sequences(me_gpu, port, seed):
    c = _fuzz_case(1000 + seed)
    from backends import GpuBackend, PortBackend

    kw = dict(halfpel=c["halfpel"], ref_distance=c["ref_distance"], bt=c["bt"], max_iter=c["max_iter"], step=c["step"], eps=c["eps"], theta=c["theta"])
    got_r, got_s = GpuBackend().run_sequence(c["algo"], c["luma"], c["alpha"], c["bs"], c["S"], **kw)
    want_r, want_s = PortBackend().run_sequence(c["algo"], c["luma"], c["alpha"], c["bs"], c["S"], **kw)
    assert_recs(got_r, want_r, f"fuzz {seed}: { {k: v for k, v in c.items() if k not in ('luma', 'alpha')} }")
    assert np.array_equal(got_s, want_s)


def _fuzz_batch(seed):
    """A batch of sequences sharing geometry and configuration (_fuzz_case's
    draws), with binary masks more often so the bit-plane path is covered."""
    rng = np.random.default_rng(5000 + seed)
    c = _fuzz_case(7000 + seed)
    n_seq = int(rng.integers(2, 6))
    F, H, W = c["luma"].shape
    lumas, alphas = [c["luma"]], [c["alpha"]]
    for i in range(1, n_seq):
        ci = _fuzz_case(9000 + 100 * seed + i)
        li = ci["luma"]
        # same geometry: crop / tile the other case's content to (F, H, W)
        li = np.resize(li, (F,) + li.shape[1:])
        li = np.tile(li, (1, (H + li.shape[1] - 1) // li.shape[1], (W + li.shape[2] - 1) // li.shape[2]))[:, :H, :W]
        lumas.append(np.ascontiguousarray(li))
        if c["alpha"] is not None:
            a = np.zeros((F, H, W), np.uint8)
            for t in range(F):
                x0, y0 = int(rng.integers(0, W // 2)), int(rng.integers(0, H // 2))
                a[t, y0:y0 + int(rng.integers(4, H)), x0:x0 + int(rng.integers(4, W))] = 255
            if rng.random() < 0.3:
                a[:, rng.integers(0, H, 3), rng.integers(0, W, 3)] = 77
            alphas.append(a)
    luma = np.stack(lumas)
    alpha = None if c["alpha"] is None else np.stack(alphas)
    return c, luma, alpha


@pytest.mark.parametrize("seed", range(150))
def test_fuzz_batches(me_gpu, port, seed):
    """Whole batches through every batched entry point (host buffers, device
    bytes, device bit planes when the masks are binary) and, for PA, a random
    kernel schedule, each against the oracle sequence by sequence."""
    import torch

    from paper_1002_1168_b200 import _lib, batch as B

    c, luma, alpha = _fuzz_batch(seed)
    me = me_gpu
    cfg = me.BatchConfig(algo=me.Algo(c["algo"]), search=me.SearchConfig(search_range=c["S"], block_size=c["bs"], ref_distance=c["ref_distance"], halfpel=bool(c["halfpel"])),
                         prs=me.PrsConfig(epsilon=c["eps"], theta=c["theta"], max_iterations=c["max_iter"], step=c["step"]), boundary_temporal=me.BoundaryTemporal(c["bt"]))
    kw = dict(halfpel=c["halfpel"], ref_distance=c["ref_distance"], bt=c["bt"], max_iter=c["max_iter"], step=c["step"], eps=c["eps"], theta=c["theta"])
    from backends import PortBackend

    want = [PortBackend().run_sequence(c["algo"], luma[i], None if alpha is None else alpha[i], c["bs"], c["S"], **kw) for i in range(len(luma))]
    what = f"batch fuzz {seed}: n_seq {len(luma)} { {k: v for k, v in c.items() if k not in ('luma', 'alpha')} }"
    rng = np.random.default_rng(seed)
    sched = str(rng.choice(["auto", "warp", "fast", "duo", "duo-hybrid", "hybrid"])) if c["algo"] == 4 else "auto"
    prev = _lib.set_tuning(0, pa_schedule=sched, pa_static_claim=int(rng.random() < 0.2), pa_key_plain=int(rng.integers(-1, 2)))
    try:
        recs, stats = me.run_sequences(cfg, luma, alpha)
        dl = torch.from_numpy(luma).cuda()
        da = None if alpha is None else torch.from_numpy(alpha).cuda()
        r_dev, s_dev = B.run_sequences_dev(cfg, dl, da)
        sv = lambda t: t.cpu().numpy().view(stats.dtype).reshape(stats.shape)  # noqa: E731
        outs = [("host", recs, stats), ("dev", B.rec_view(r_dev), sv(s_dev))]
        if da is not None:
            bits, binary = B.pack_mask_dev(da)
            if binary:
                r_b, s_b = B.run_sequences_bits_dev(cfg, dl, bits)
                outs.append(("bits", B.rec_view(r_b), sv(s_b)))
        torch.cuda.synchronize()
    finally:
        _lib.restore_tuning(prev, 0)
    for name, r, s in outs:
        for i, (wr, ws) in enumerate(want):
            assert_recs(r[i].reshape(wr.shape), wr, f"{what} [{name}, sched {sched}, seq {i}]")
            assert np.array_equal(s[i].reshape(ws.shape), ws), f"{what} [{name}] stats seq {i}"
