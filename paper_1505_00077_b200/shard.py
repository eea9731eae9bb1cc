"""Frame sharding across GPUs: one process per GPU, frames
partitioned contiguously, no collective on the data path.

Every frame of a batch or video channel is an independent problem -- the
recursive Gaussian's unbounded support never crosses a frame -- so a batch of
F frames is split into contiguous blocks, rank r filtering frames
[start_r, stop_r) on its own device. Only scalars cross ranks, on the host
side of the timed region: the per-rank time (max over ranks, the job's time)
and the per-frame fallback counts (each frame's count is owned by the rank
that filtered it).
"""
from __future__ import annotations

from typing import Callable, Sequence


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of `n_items` for `rank` of `world`; block sizes differ
    by at most one, the larger blocks first."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    if n_items < 0:
        raise ValueError("n_items must be >= 0")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(n_items: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_range(n_items, r, world) for r in range(world))]


def reduce_job(local_seconds: float, local_fallbacks: Sequence[int], n_items: int, rank: int,
               world: int, device=None) -> tuple[float, list[int]]:
    """Host-side reduction after the timed region: the job time is the max over
    ranks, the fallback list is assembled in frame order. With world == 1 no
    process group is needed."""
    start, stop = shard_range(n_items, rank, world)
    if len(local_fallbacks) != stop - start:
        raise ValueError("one fallback count per local frame expected")
    if world == 1:
        return float(local_seconds), [int(v) for v in local_fallbacks]
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local_seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    fb = torch.zeros(n_items, dtype=torch.int64, device=device)
    fb[start:stop] = torch.tensor([int(v) for v in local_fallbacks], dtype=torch.int64)
    dist.all_reduce(fb, op=dist.ReduceOp.SUM)  # disjoint blocks: a sum is an assembly
    return float(t.item()), [int(v) for v in fb.cpu().tolist()]


def run_shard(frames, rank: int, world: int, filter_fn: Callable):
    """Filters this rank's block of `frames` (indexable, len() = frame count) with
    `filter_fn(block) -> (out_block, fallbacks)`. Returns (start, out, fallbacks)."""
    start, stop = shard_range(len(frames), rank, world)
    out, fb = filter_fn(frames[start:stop])
    return start, out, list(fb)
