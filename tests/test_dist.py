"""Multi-rank host logic on CPU (gloo, world size 2): sharding, seeds and the
final MV-field gather the GPU bench does over NCCL."""
import os
import socket

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
