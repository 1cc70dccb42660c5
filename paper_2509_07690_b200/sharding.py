"""Batch sharding for the batched refactorization workload.

Independent same-pattern instances are split contiguously across ranks; each
rank uploads the symbolic structure once and processes its slab.  There is no
collective on the data path; the only cross-rank operations are the max-over-ranks
of the timed region and an optional result gather off the clock.
"""

from __future__ import annotations

import numpy as np


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


def all_values(value, dist=None, device=None):
    """Every rank's float, in rank order (per-rank device times for the report)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(value)]
    import torch
    w = dist.get_world_size()
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(w)]
    dist.all_gather(out, t)
    return [float(o.item()) for o in out]


def gather_shards(local, total, dist=None, device=None):
    """Assemble the [total, ...] result from every rank's contiguous shard (off the
    clock; ``local`` is a numpy array of the rank's rows).  Returns the full array
    on every rank."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return np.asarray(local)
    import torch
    w, r = dist.get_world_size(), dist.get_rank()
    lo, hi = shard_range(total, r, w)
    if local.shape[0] != hi - lo:
        raise ValueError("shard has %d rows, expected %d" % (local.shape[0], hi - lo))
    width = max(hi2 - lo2 for lo2, hi2 in (shard_range(total, k, w) for k in range(w)))
    pad = np.zeros((width,) + local.shape[1:], local.dtype)
    pad[:hi - lo] = local
    t = torch.from_numpy(pad).to(device) if device is not None else torch.from_numpy(pad)
    out = [torch.empty_like(t) for _ in range(w)]
    dist.all_gather(out, t)
    parts = []
    for k in range(w):
        lo2, hi2 = shard_range(total, k, w)
        parts.append(out[k].cpu().numpy()[:hi2 - lo2])
    return np.concatenate(parts, axis=0)
