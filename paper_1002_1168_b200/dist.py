"""Multi-GPU plumbing for the batched pipeline.

The work shards with no data-path collective: configuration 4's 256
independent sequences (and the baselines' frame pairs) are split across ranks,
one process per GPU.  The only collective is the final gather of the
motion-vector fields into rank 0 (torch.distributed over NCCL/NVLink on B200,
gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def coll_device(device, group=None):
    """Where collective buffers live: `device` under NCCL, the host under gloo
    (the CPU tests, and the bench's one-GPU multi-rank check)."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return device


def shard(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced split of n_total units: (first, count) of `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def sequence_seeds(base_seed: int, per_rank: int, rank: int, world: int, strong: bool = False, n_total: Optional[int] = None) -> List[int]:
    """Seeds of this rank's sequences (config 4: seed = base + i).

    weak scaling: every rank runs its own `per_rank` sequences
    (global indices rank * per_rank + i); strong scaling: the n_total
    sequences are sharded."""
    if strong:
        first, count = shard(n_total if n_total is not None else per_rank, rank, world)
        return [base_seed + first + i for i in range(count)]
    return [base_seed + rank * per_rank + i for i in range(per_rank)]


def mv_words(recs):
    """The int32 motion-vector words (dx | dy << 16) of a uint8 record tensor
    [..., 16] as a contiguous tensor [...] (a strided view, then a copy)."""
    import torch

    return recs.view(torch.int32)[..., 0].contiguous()


def gather_fields(mv, dst: int = 0, group=None):
    """Gathers every rank's MV-word tensor into rank `dst` (None elsewhere).
    Tensors must have the same shape on every rank."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [mv]
    rank = dist.get_rank(group)
    out = [torch.empty_like(mv) for _ in range(dist.get_world_size(group))] if rank == dst else None
    dist.gather(mv, out, dst=dst, group=group)
    return out


def pack_mv(recs, search_range: int):
    """The MV field of a uint8 record tensor [..., 16] in its smallest exact
    form: (dx, dy) as int8 pairs [..., 2] when every vector fits (half-pel
    components lie in [-2S, 2S], so S <= 63), else the int32 words of
    `mv_words`.  One elementwise pass over the records."""
    import torch

    if 2 * search_range <= 127:
        return recs.view(torch.int16)[..., 0:2].to(torch.int8)
    return mv_words(recs)


def unpack_mv(packed):
    """(dx, dy) int32 [..., 2] from either `pack_mv` form."""
    import torch

    if packed.dtype == torch.int8:
        return packed.to(torch.int32)
    return torch.stack([(packed << 16) >> 16, packed >> 16], dim=-1)


class FieldGatherer:
    """Per-step gather of the MV fields into rank `dst`, overlapped with the
    next step: step k's packed field is gathered asynchronously (NCCL runs it
    on its own stream after step k's kernels) while step k+1 computes; two
    send buffers alternate (a buffer is refilled only after its previous
    gather completed, `Work.wait`, a stream dependency under NCCL), and the
    receive buffers rotate through three sets, so `fields` — the latest
    COMPLETED step's fields on rank `dst` — is never the target of a gather in
    flight.  `finish` waits for the last gather."""

    def __init__(self, search_range: int, dst: int = 0, group=None):
        self.S, self.dst, self.group = search_range, dst, group
        self.bufs = [None, None]
        self.outs = [None, None, None]
        self.slot = [0, 0]
        self.work = [None, None]
        self.k = 0
        self.fields = None

    def submit(self, recs):
        import torch
        import torch.distributed as dist

        i = self.k & 1
        if self.work[i] is not None:
            self.work[i].wait()
            self.fields = self.outs[self.slot[i]]
        packed = pack_mv(recs, self.S)
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        if self.bufs[i] is None or self.bufs[i].shape != packed.shape or self.bufs[i].dtype != packed.dtype:
            self.bufs[i] = torch.empty_like(packed)
            self.outs = [None, None, None]
        j = self.k % 3
        if rank == self.dst and self.outs[j] is None:
            self.outs[j] = [torch.empty_like(packed) for _ in range(world)]
        self.bufs[i].copy_(packed)
        self.slot[i] = j
        self.work[i] = dist.gather(self.bufs[i], self.outs[j] if rank == self.dst else None, dst=self.dst, group=self.group, async_op=True)
        self.k += 1

    def finish(self):
        """Waits for every outstanding gather; returns rank dst's fields of
        the last step (None on the other ranks)."""
        for j in (self.k & 1, (self.k + 1) & 1):  # older first
            if self.work[j] is not None:
                self.work[j].wait()
                self.fields = self.outs[self.slot[j]]
                self.work[j] = None
        return self.fields


class ResultGatherer:
    """Per-step gather of every rank's results into rank `dst`, overlapped with
    the next step ("int64 SSE gathered with the records"): the
    packed MV field (`pack_mv`) and the per-pair SearchStats + SSE (48 bytes
    per pair) of a rank's `counts[rank]` sequences go in ONE uint8 buffer,
    padded to the largest shard (a gather needs equal sizes), gathered
    asynchronously on the collective's stream while the next step computes.
    Send buffers alternate (a buffer is refilled only after its previous gather
    completed) and the received buffers rotate through three sets, so the
    result of the latest completed step stays valid until two more steps have
    been submitted."""

    def __init__(self, search_range: int, counts: List[int], dst: int = 0, group=None):
        self.S, self.counts, self.dst, self.group = search_range, list(counts), dst, group
        self.nmax = max(self.counts)
        self.send = [None, None]
        self.recv = [None, None, None]
        self.work = [None, None]
        self.slot = [0, 0]  # recv set used by the gather in flight from send buffer i
        self.k = 0
        self.done_slot = None
        self.layout = None

    def _pack(self, recs, stats):
        import torch

        mv = pack_mv(recs, self.S)
        n = recs.shape[0]
        mvb = mv.reshape(n, -1).view(torch.uint8) if mv.dtype == torch.int8 else mv.reshape(n, -1).contiguous().view(torch.uint8)
        stb = stats.reshape(n, -1)
        if self.layout is None:
            self.layout = (mv.dtype, tuple(mv.shape[1:]), mvb.shape[1], stb.shape[1], tuple(stats.shape[1:]))
        return mvb, stb

    def submit(self, recs, stats):
        import torch
        import torch.distributed as dist

        i = self.k & 1
        if self.work[i] is not None:
            self.work[i].wait()
            self.done_slot = self.slot[i]
        mvb, stb = self._pack(recs, stats)
        per = mvb.shape[1] + stb.shape[1]
        if self.send[i] is None:
            self.send[i] = torch.zeros((self.nmax, per), dtype=torch.uint8, device=coll_device(recs.device, self.group))
        n = recs.shape[0]
        self.send[i][:n, : mvb.shape[1]].copy_(mvb)
        self.send[i][:n, mvb.shape[1]:].copy_(stb)
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        j = self.k % 3
        if rank == self.dst and self.recv[j] is None:
            self.recv[j] = [torch.empty_like(self.send[i]) for _ in range(world)]
        self.slot[i] = j
        self.work[i] = dist.gather(self.send[i], self.recv[j] if rank == self.dst else None, dst=self.dst, group=self.group, async_op=True)
        self.k += 1

    def finish(self):
        """Waits for every outstanding gather; on rank dst returns the last
        completed step's (mv [n_total, pairs, rows, cols, 2] int32,
        stats [n_total, pairs, 48] uint8) in rank order, else None."""
        import torch
        import torch.distributed as dist

        for j in (self.k & 1, (self.k + 1) & 1):  # older first
            if self.work[j] is not None:
                self.work[j].wait()
                self.done_slot = self.slot[j]
                self.work[j] = None
        if dist.get_rank(self.group) != self.dst or self.done_slot is None:
            return None
        dtype, mvshape, mvbytes, stbytes, stshape = self.layout
        mvs, sts = [], []
        for r, buf in enumerate(self.recv[self.done_slot]):
            n = self.counts[r]
            m = buf[:n, :mvbytes]
            m = m.view(torch.int8) if dtype == torch.int8 else m.contiguous().view(torch.int32)
            mvs.append(unpack_mv(m.reshape((n,) + mvshape)))
            sts.append(buf[:n, mvbytes: mvbytes + stbytes].reshape((n,) + stshape))
        return torch.cat(mvs), torch.cat(sts)


def band_units(alpha, bs: int, pairs: int, d: int, n_bands: int):
    """The baselines' sharding units: (band, pair) with the block
    rows split into n_bands bands, each with its estimated-block count (the
    work a unit costs: transparent blocks are skipped, estimators.cpp:418).
    `alpha` is one sequence's [F, H, W] uint8 tensor (any device); a block is
    estimated unless its CURRENT alpha (frame p + d) is all zero
    (classify_block, frame.cpp:81-104).  Returns [(band, pair, row0, row1,
    estimated)] band-major."""
    import numpy as np
    import torch

    F, H, W = alpha.shape
    rows, cols = H // bs, W // bs
    cur = alpha[d:d + pairs].reshape(pairs, rows, bs, cols, bs)
    est = (cur.amax(dim=(2, 4)) > 0).to(torch.int64)
    per_row = est.sum(dim=2).cpu().numpy()  # [pairs, rows]
    edges = np.linspace(0, rows, n_bands + 1).round().astype(int)
    return [(b, p, int(edges[b]), int(edges[b + 1]), int(per_row[p, edges[b]:edges[b + 1]].sum()))
            for b in range(n_bands) for p in range(pairs)]


def split_units(units, world: int):
    """Contiguous split of the (band-major) units over `world` ranks, balanced
    by estimated-block count (+1 per unit for its fixed cost)."""
    import numpy as np

    cost = np.array([u[4] + 1 for u in units], dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    cuts = [0] + [int(np.searchsorted(cum, cum[-1] * r / world)) for r in range(1, world)] + [len(units)]
    return [units[cuts[r]:cuts[r + 1]] for r in range(world)]


def unit_runs(units):
    """A rank's units grouped into calls: [band, first pair, end pair, row0,
    row1] for runs of consecutive pairs of one band (one me_b200_run_band_dev
    call each: the pairs are a frame sub-range of the sequence)."""
    runs = []
    for b, p, r0, r1, _ in units:
        if runs and runs[-1][0] == b and runs[-1][2] == p:
            runs[-1][2] = p + 1
        else:
            runs.append([b, p, p + 1, r0, r1])
    return runs


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timings: the slowest rank defines the job)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
