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


# ---------------------------------------------------------------------------
# Row-partitioned tree construction.
#
# The complete tree over I rows (leaf capacity F = R, init_tree
# segment_tree_sampler.cpp:111-149) splits into parts = 2^g subtrees, the nodes
# of level g. Compact slot s >= 1 stores heap node 2s-1, so the stored nodes of
# tree level l are the slot range [2^(l-1), 2^l) and, for every level below g,
# subtree i owns an equal contiguous sub-range of it (the leaf level d of a
# non-perfect tree is ragged: ranges are padded to equal size for the
# exchange). Each rank builds its subtree (krpg_build_partition), the per-level
# ranges and the subtree roots are all-gathered, and the top g levels are
# reduced redundantly on every rank (krpg_finish_partitions).
# ---------------------------------------------------------------------------
def _ceil_log2(x: int) -> int:
    return 0 if x <= 1 else (x - 1).bit_length()


def tree_geometry(I: int, R: int) -> dict:
    """Leaf count L, depth d, positions npos (level d-1 nodes), hb (positions that
    are pairs of depth-d leaves)."""
    L = (I + R - 1) // R
    d = _ceil_log2(L)
    bottom = 2 * L - (1 << d)
    npos = 1 << (d - 1) if d >= 1 else 1
    return {"L": L, "d": d, "bottom": bottom, "npos": npos, "hb": bottom // 2}


def partition_slots(I: int, R: int, parts: int, part: int) -> list[tuple[int, int, int, int]]:
    """Exchange plan of subtree `part` of `parts`: a list of
    (level, level_slot0, span, valid) -- on tree level `level`, the rank owns the
    compact slots [level_slot0 + part*span, level_slot0 + part*span + valid);
    every rank's range has the padded size `span`, and the level's slots are
    [level_slot0, level_slot0 + parts*span) clipped to the tree (L slots)."""
    geo = tree_geometry(I, R)
    d, npos, hb, L = geo["d"], geo["npos"], geo["hb"], geo["L"]
    if parts < 2 or parts & (parts - 1) or parts > npos:
        raise ValueError("partition_slots: parts must be a power of two in [2, positions]")
    if not 0 <= part < parts:
        raise ValueError("partition_slots: part out of range")
    g = parts.bit_length() - 1
    plan = []
    for lev in range(g + 1, d):  # internal / position levels: 2^(lev-1) stored slots
        span = (1 << (lev - 1)) // parts
        plan.append((lev, 1 << (lev - 1), span, span))
    if d >= 1 and hb > 0:  # leaf level d: left leaves of the pair positions j < hb
        span = npos // parts
        p0 = part * span
        valid = max(0, min(p0 + span, hb) - p0)
        plan.append((d, 1 << (d - 1), span, valid))
    assert all(s0 + parts * sp <= L or lev == d for lev, s0, sp, _ in plan)
    return plan


def exchange_partitioned_tree(tree, subroot, I: int, R: int, group=None):
    """All-gather a row-partitioned tree in place.

    ``tree``: flat tensor of L*P doubles holding this rank's owned slots (others
    are overwritten); ``subroot``: this rank's subtree root Gram (P doubles).
    Returns the parts x P tensor of all subtree roots (input of
    krpg_finish_partitions). Works over any torch.distributed backend (NCCL on
    device tensors, gloo on host tensors); rank r of the group owns subtree r."""
    import torch
    import torch.distributed as dist
    parts = dist.get_world_size(group)
    part = dist.get_rank(group)
    P = R * (R + 1) // 2
    L = tree_geometry(I, R)["L"]
    for lev, s0, span, _valid in partition_slots(I, R, parts, part):
        n = span * P
        mine = tree[(s0 + part * span) * P:(s0 + part * span) * P + n].clone() \
            if (s0 + part * span) * P + n <= L * P else _padded(tree, (s0 + part * span) * P, n, L * P)
        out = torch.empty(parts * n, dtype=tree.dtype, device=tree.device)
        dist.all_gather_into_tensor(out, mine, group=group)
        end = min(L * P, (s0 + parts * span) * P)
        tree[s0 * P:end] = out[:end - s0 * P]
    roots = torch.empty(parts * P, dtype=subroot.dtype, device=subroot.device)
    dist.all_gather_into_tensor(roots, subroot.contiguous(), group=group)
    return roots


def _padded(tree, start: int, n: int, total: int):
    import torch
    out = torch.zeros(n, dtype=tree.dtype, device=tree.device)
    have = max(0, min(total, start + n) - start)
    if have:
        out[:have] = tree[start:start + have]
    return out


class _DeviceArray:
    """Zero-copy view of device memory owned by the sampler (for torch collectives)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def build_partitioned(sampler, j: int, group=None) -> None:
    """Rebuild factor j's tree with the rows split over the ranks of `group`
    (one process per GPU, NCCL): every rank builds its subtree from its rows of
    U_j, then the stored slots and subtree roots are all-gathered and the top
    levels reduced locally. U_j must hold at least this rank's rows on every
    rank (all-gather the factor first when it is row-partitioned)."""
    import torch
    import torch.distributed as dist
    parts, part = dist.get_world_size(group), dist.get_rank(group)
    I, R = int(sampler._dims[j]), int(sampler._R)
    P = R * (R + 1) // 2
    tree = sampler.tree_device(j)
    subroot = torch.empty(P, dtype=torch.float64, device="cuda")
    sampler.build_partition(j, parts, part, subroot)
    roots = exchange_partitioned_tree(tree, subroot, I, R, group)
    torch.cuda.synchronize()
    sampler.finish_partitions(j, parts, roots)
