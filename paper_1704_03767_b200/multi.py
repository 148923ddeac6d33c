"""Multi-GPU plumbing: one process per GPU, contiguous job-id shards, optional gather.

Every pair is independent, so ranks never exchange data while computing:
rank r of p computes job ids ``job_shard_range(r, p, m)`` (the reference's
contiguous ceil-chunk shard rule, pairindex.py:68-80, applied to job ids), and
the shards concatenate to the full job-id stream.  The only collective is the
optional gather of result shards to one consumer rank -- an all_gather of
equal, padded chunks (NCCL over NVLink on a B200 box; gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .pairindex import job_shard_range


def my_job_range(m: int, rank: int | None = None, world: int | None = None) -> tuple[int, int]:
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return job_shard_range(rank, world, m)


def gather_shards(local: torch.Tensor, m: int, dst: int = 0, group=None) -> torch.Tensor | None:
    """Concatenate every rank's job-range shard on rank ``dst`` (None elsewhere).

    ``local`` is this rank's per-pair tensor for ``my_job_range(m)``.  Shards
    are padded to the common chunk length so one all_gather_into_tensor moves
    them; ``dst`` trims the padding.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = m * (m + 1) // 2
    chunk = -(-total // world)
    lo, hi = job_shard_range(rank, world, m)
    if local.numel() != hi - lo:
        raise ValueError(f"rank {rank}: shard has {local.numel()} entries, expected {hi - lo}")
    padded = torch.zeros(chunk, dtype=local.dtype, device=local.device)
    padded[: local.numel()] = local
    out = torch.empty(chunk * world, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        a, b = job_shard_range(r, world, m)
        parts.append(out[r * chunk: r * chunk + (b - a)])
    return torch.cat(parts)
