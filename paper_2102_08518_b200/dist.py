"""Multi-GPU plumbing for the query-sharded evaluator.

Queries are independent, so N GPUs split the global query index range and
each evaluates its shard against a full replica of the coefficient volume:
no collective in the evaluation loop.  The only communication is one
broadcast of the volume from rank 0 at setup (NCCL over NVLink on the GPU
box, gloo in the CPU tests) and the max-over-ranks reduction of timings.
"""

from __future__ import annotations

import numpy as np


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous [lo, hi) slice of the global query index for `rank`."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def replicate_arrays(arrays, device=None, src: int = 0):
    """Broadcast rank `src`'s coset arrays to every rank (torch.distributed must be
    initialized).  Returns torch tensors on `device` (CPU for gloo)."""
    import torch
    import torch.distributed as dist
    out = []
    for a in arrays:
        t = torch.as_tensor(np.ascontiguousarray(a))
        if device is not None:
            t = t.to(device)
        dist.broadcast(t, src)
        out.append(t)
    return out


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local, n_total: int, device=None):
    """Optional result gather to every rank (all_gather of equal-size padded shards)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    per = -(-n_total // world)
    buf = torch.zeros(per, dtype=local.dtype, device=device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        out.append(parts[r][: hi - lo])
    return torch.cat(out)
