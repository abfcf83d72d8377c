"""Multi-GPU plumbing for the batched pipeline.

The work shards with no data-path collective: configuration 4's 256
independent sequences (and the baselines' frame pairs) are split across ranks,
one process per GPU.  The only collective is the final gather of the
motion-vector fields into rank 0 (torch.distributed over NCCL/NVLink on B200,
gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Optional, Tuple


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


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timings: the slowest rank defines the job)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
