"""Multi-GPU draw sharding.

Draws are independent and every draw's uniforms are keyed by its global draw
index (CounterRng stream = draw id, rng.hpp:13-48 / krp_sampler.cpp:107-109),
so J draws split across ranks as contiguous ranges [start, start+count) with
``draw_offset = start`` reproduce one big call exactly. No collective is on
the data path; a gather is only needed when one rank wants all draws.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_range(J: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of J draws: (start, count) for this rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    base, rem = divmod(J, world)
    start = rank * base + min(rank, rem)
    count = base + (1 if rank < rem else 0)
    return start, count


def sample_sharded(sample_fn: Callable, excluded: Optional[int], J: int, seed: int, rank: int,
                   world: int, group=None, gather: bool = True):
    """Draw this rank's share of J samples; optionally all-gather to every rank.

    ``sample_fn(excluded, count, seed, draw_offset)`` -> (idx, prob, rows) numpy
    arrays (e.g. ``KrpSampler.sample`` or an oracle). The gather runs over
    torch.distributed (gloo for CPU tests, NCCL on GPUs)."""
    start, count = shard_range(J, rank, world)
    idx, prob, rows = sample_fn(excluded, count, seed, start)
    if not gather or world == 1:
        return idx, prob, rows
    import torch
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, (start, idx, prob, rows), group=group)
    parts.sort(key=lambda p: p[0])
    return (np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts]),
            np.concatenate([p[3] for p in parts]))
