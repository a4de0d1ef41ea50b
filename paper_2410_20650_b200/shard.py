"""Multi-GPU partitioning of the codec path (host logic, no collectives on
the data path).

The path partitions naturally: every tensor has its own frequency table
(tensorstore.hpp:103, :203) and, given the table, chunks are independent
(ans.hpp:258-271).  So a model is sharded by whole tensors; each rank owns
its tensors' compressed bytes in its own HBM and decodes them locally.  The
only cross-rank communication is plumbing: agreeing on the assignment
(deterministic, so no communication at all) and reducing the timing /
byte counts for reporting (max over ranks, sum of bytes).
"""
from __future__ import annotations

import heapq
from typing import Sequence


def lpt_assign(sizes: Sequence[int], world: int) -> list:
    """Longest-processing-time-first assignment of tensors to ranks by
    element count.  Deterministic (ties broken by tensor index, then by rank),
    so every rank computes the same plan without communicating.
    Returns rank-of-tensor."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    heap = [(0, r) for r in range(world)]
    owner = [0] * len(sizes)
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return owner


def shard_loads(sizes: Sequence[int], owner: Sequence[int], world: int) -> list:
    loads = [0] * world
    for s, r in zip(sizes, owner):
        loads[r] += int(s)
    return loads


def imbalance(sizes: Sequence[int], world: int) -> float:
    """max-load / mean-load of the LPT plan (1.0 = perfect)."""
    loads = shard_loads(sizes, lpt_assign(sizes, world), world)
    mean = sum(loads) / world
    return max(loads) / mean if mean else 1.0


def reduce_timing(dist, elapsed_s: float, bytes_local: int, device=None):
    """All ranks -> (max elapsed, total bytes): the whole-job throughput is
    sum(bytes) / max(time).  `dist` is torch.distributed (any backend)."""
    import torch

    t = torch.tensor([elapsed_s], dtype=torch.float64, device=device)
    b = torch.tensor([float(bytes_local)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    return float(t.item()), int(b.item())
