"""Replica sharding for N GPUs (one process per GPU).

The DART tree and the wave semantics are not splittable, so the path scales as
independent replicas: requests are routed by a hash of their first skeleton
segment and each GPU runs its own QAS + DART on its
sub-trace.  The only exchange is one all-reduce (sum) per scheduling window of
the per-segment demand counters (NCCL over NVLink on GPUs; gloo in the CPU
tests), plus max-over-ranks timing.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64."""
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(_M64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def route(first_segments: Sequence[int] | np.ndarray, world: int) -> np.ndarray:
    """Shard of each request: splitmix64(skeleton[0]) mod world."""
    a = np.asarray(first_segments, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return (splitmix64(a) % np.uint64(world)).astype(np.int64)


def shard_requests(requests: Sequence, world: int, rank: int) -> list:
    """The requests of one replica, in their original order."""
    if not requests:
        return []
    firsts = np.array([r.skeleton[0] if r.skeleton else -1 for r in requests], dtype=np.int64)
    firsts = np.where(firsts < 0, 0, firsts)
    sh = route(firsts, world)
    return [r for r, s in zip(requests, sh.tolist()) if s == rank]


def allreduce_demand(counts, group=None):
    """Sum the per-window demand counter vector over all replicas (in place)."""
    import torch.distributed as dist

    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def max_over_ranks(value: float, device=None) -> float:
    """The job's time is the slowest replica's (bench timing rule)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
