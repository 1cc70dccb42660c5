"""Batch sharding for the batched refactorization workload.

Independent same-pattern instances are split contiguously across ranks; each
rank uploads the symbolic structure once and processes its slab.  There is no
collective on the data path; the only cross-rank operation is the max-over-ranks
of the timed region (and an optional result gather off the clock).
"""

from __future__ import annotations


def shard_range(total, rank, world):
    """Contiguous [lo, hi) slab of ``total`` instances owned by ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return rank * total // world, (rank + 1) * total // world


def max_over_ranks(value, dist=None, device=None):
    """Max of a float over all ranks (device time of the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
