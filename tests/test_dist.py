"""Multi-rank host logic on CPU (gloo, world size 2): sharding, seeds and the
final MV-field gather the GPU bench does over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1002_1168_b200 import dist as mdist


def test_shard_covers_everything():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            spans = [mdist.shard(n, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == n
            pos = 0
            for first, count in spans:
                assert first == pos
                pos += count
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        mdist.shard(4, 2, 2)


def test_pack_mv_both_forms():
    recs = torch.zeros((3, 7, 16), dtype=torch.uint8)
    r16 = recs.view(torch.int16)
    r16[..., 0] = torch.arange(-10, 11, dtype=torch.int16).view(3, 7) * 6  # up to +-60
    r16[..., 1] = -torch.arange(-10, 11, dtype=torch.int16).view(3, 7) * 3
    want = r16[..., 0:2].to(torch.int32)
    small = mdist.pack_mv(recs, 31)
    assert small.dtype == torch.int8 and torch.equal(mdist.unpack_mv(small), want)
    r16[..., 0] *= 2  # up to +-120 half-pel: S = 64 needs the int32 words
    want = r16[..., 0:2].to(torch.int32)
    wide = mdist.pack_mv(recs, 64)
    assert wide.dtype == torch.int32 and torch.equal(mdist.unpack_mv(wide), want)


def test_seeds_weak_and_strong():
    weak = [mdist.sequence_seeds(100, 4, r, 2) for r in range(2)]
    assert weak == [[100, 101, 102, 103], [104, 105, 106, 107]]
    strong = [mdist.sequence_seeds(100, 0, r, 3, strong=True, n_total=8) for r in range(3)]
    assert sum(strong, []) == list(range(100, 108))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # fake per-rank record batch [seq, pair, rows, cols, 16]; MV word = rank-tagged
        recs = torch.zeros((2, 3, 4, 5, 16), dtype=torch.uint8)
        w = recs.view(torch.int32)
        w[..., 0] = torch.arange(2 * 3 * 4 * 5, dtype=torch.int32).view(2, 3, 4, 5) + 1000 * rank
        got = mdist.gather_fields(mdist.mv_words(recs))
        # the pipelined compact gather: 3 steps, each with its own field
        g = mdist.FieldGatherer(search_range=16)
        for step in range(3):
            r16 = recs.view(torch.int16)
            r16[..., 0] = (torch.arange(120, dtype=torch.int16).view(2, 3, 4, 5) % 65) - 32 + step
            r16[..., 1] = -(torch.arange(120, dtype=torch.int16).view(2, 3, 4, 5) % 61) + 30 + rank
            want_step = mdist.unpack_mv(mdist.pack_mv(recs, 16)).clone()
            g.submit(recs)
        last = g.finish()
        if rank == 0:
            assert len(last) == 2
            assert torch.equal(mdist.unpack_mv(last[0]), want_step)
            assert torch.equal(mdist.unpack_mv(last[1])[..., 0], want_step[..., 0])
            assert torch.equal(mdist.unpack_mv(last[1])[..., 1], want_step[..., 1] + 1)
        else:
            assert last is None
        t = mdist.max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put(([g.tolist() for g in got], t))
        else:
            assert got is None
            q.put(None)
    finally:
        dist.destroy_process_group()


def test_gather_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fields, tmax = next(r for r in results if r is not None)
    assert tmax == 2.0
    base = torch.arange(120, dtype=torch.int32).view(2, 3, 4, 5)
    assert fields[0] == base.tolist()
    assert fields[1] == (base + 1000).tolist()


# ---------------------------------------------------------------------------
# The bench's multi-GPU paths, host logic on CPU: each rank's compute is the
# oracle restatement (a CPU stand-in for the CUDA path), the plumbing is the
# product's (paper_1002_1168_b200.dist) over gloo.

def _recs_tensor(recs_np, stats_np):
    """numpy record/stat arrays -> the uint8 tensors the CUDA path produces."""
    r = torch.from_numpy(np.ascontiguousarray(recs_np).view(np.uint8).reshape(recs_np.shape + (16,)))
    s = torch.from_numpy(np.ascontiguousarray(stats_np).view(np.uint8).reshape(stats_np.shape + (48,)))
    return r, s


def _strong_worker(rank, world, port, q, n_total, frames):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1002_1168_b200 import synth

        counts = [mdist.shard(n_total, r, world)[1] for r in range(world)]
        first, n = mdist.shard(n_total, rank, world)
        luma, alpha = synth.config4_batch(n, 900 + first, frames, threads=2)
        port = oracle.Oracle("port")
        cfg = oracle.make_cfg(algo=4, search_range=16, block_size=8)
        out = [port.run_sequence(cfg, luma[i], alpha[i]) for i in range(n)]
        recs, stats = _recs_tensor(np.stack([o[0] for o in out]), np.stack([o[1] for o in out]))
        g = mdist.ResultGatherer(16, counts)
        for _ in range(3):  # three steps in flight, like the bench
            g.submit(recs, stats)
        res = g.finish()
        q.put(None if res is None else (res[0].numpy(), res[1].numpy()))
    finally:
        dist.destroy_process_group()


def test_strong_sharded_config4_gloo():
    """config 4 strong-sharded over 2 ranks (5 sequences: 3 + 2), per-step
    gather of MV fields + stats/SSE: rank 0's merged result equals a 1-rank
    run over the whole batch."""
    import oracle
    from paper_1002_1168_b200 import synth

    n_total, frames = 5, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, 2, port, q, n_total, frames)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mv, st = next(r for r in results if r is not None)
    luma, alpha = synth.config4_batch(n_total, 900, frames, threads=2)
    po = oracle.Oracle("port")
    cfg = oracle.make_cfg(algo=4, search_range=16, block_size=8)
    want = [po.run_sequence(cfg, luma[i], alpha[i]) for i in range(n_total)]
    want_r = np.stack([w[0] for w in want])
    want_s = np.stack([w[1] for w in want])
    assert np.array_equal(mv[..., 0], want_r["dx"]) and np.array_equal(mv[..., 1], want_r["dy"])
    assert np.array_equal(st.view(want_s.dtype).reshape(want_s.shape), want_s)
    # the bench's parity digest over the gathered payload equals the one of the whole result
    rec = np.zeros(want_r.shape, want_r.dtype)
    rec["dx"], rec["dy"] = mv[..., 0], mv[..., 1]
    assert np.array_equal(oracle.digest_records(rec, want_s, 176 * 2, 144 * 2), oracle.digest_records(want_r, want_s, 352, 288))


def test_band_units_cover_and_balance():
    rng = np.random.default_rng(1)
    alpha = torch.zeros((6, 64, 96), dtype=torch.uint8)
    alpha[:, 8:40, 16:70] = 255
    alpha[2:, 48:60, 0:20] = 255
    units = mdist.band_units(alpha, 16, pairs=4, d=2, n_bands=2)
    assert len(units) == 8 and [(u[0], u[1]) for u in units] == [(b, p) for b in range(2) for p in range(4)]
    assert sum(u[4] for u in units) == int((alpha[2:].view(4, 4, 16, 6, 16).amax(dim=(2, 4)) > 0).sum())
    for world in (1, 2, 3, 8):
        parts = mdist.split_units(units, world)
        assert sum(parts, []) == units  # contiguous, every unit exactly once
    runs = mdist.unit_runs(units[1:6])
    assert runs == [[0, 1, 4, 0, 2], [1, 0, 2, 2, 4]]
    del rng


def _band_worker(rank, world, port, q):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1002_1168_b200 import synth

        luma, alpha = synth.config_sequence(1, 77, 6)  # QCIF: 4 pairs, 9 rows of 16x16 blocks
        bs, S, d = 16, 16, 2
        pairs, rows, cols = luma.shape[0] - d, luma.shape[1] // bs, luma.shape[2] // bs
        units = mdist.band_units(torch.from_numpy(alpha), bs, pairs, d, n_bands=3)
        mine = mdist.split_units(units, world)[rank]
        po = oracle.Oracle("port")
        cfg = oracle.make_cfg(algo=0, search_range=S, block_size=bs)
        mv = torch.zeros((pairs, rows, cols), dtype=torch.int32)
        for b, p0, p1, r0, r1 in mdist.unit_runs(mine):  # a frame sub-range per run, its band's rows kept
            recs, _ = po.run_sequence(cfg, luma[p0:p1 + d], alpha[p0:p1 + d])
            words = torch.from_numpy(recs.view(np.uint8).reshape(recs.shape + (16,)).copy()).view(torch.int32)[..., 0]
            mv[p0:p1, r0:r1] = words[:, r0:r1]
        got = mdist.gather_fields(mv)
        if rank == 0:
            owner = {(u[1], u[0]): (r, u[2], u[3]) for r, us in enumerate(mdist.split_units(units, world)) for u in us}
            full = torch.zeros_like(mv)
            for (p, b), (r, r0, r1) in owner.items():
                full[p, r0:r1] = got[r][p, r0:r1]
            q.put(full.numpy())
        else:
            q.put(None)
    finally:
        dist.destroy_process_group()


def test_es_band_sharding_gloo():
    """ES on (pair, row-band) units over 2 ranks: the merged MV field equals
    the 1-rank field."""
    import oracle
    from paper_1002_1168_b200 import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = next(r for r in results if r is not None)
    luma, alpha = synth.config_sequence(1, 77, 6)
    recs, _ = oracle.Oracle("port").run_sequence(oracle.make_cfg(algo=0, search_range=16, block_size=16), luma, alpha)
    want = recs.view(np.uint8).reshape(recs.shape + (16,)).copy().view(np.int32)[..., 0]
    assert np.array_equal(full, want)
