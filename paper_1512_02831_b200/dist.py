"""Multi-process (one process per GPU) helpers: query sharding and the
max-over-ranks timing reduction used by bench.py.

Queries shard naturally (reference scheduler.py:1-10, 172-183): every
query's traversal is independent and the tree is replicated, so ranks
exchange no data on the search path; the only collectives are the timing
reduction and an optional gather of results for checking.
"""
from __future__ import annotations


def shard_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Even split, remainder to the front ranks (scheduler.py:172-183)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    base, rem = divmod(m, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def max_over_ranks(x: float, device=None) -> float:
    """Maximum of a per-rank scalar (device time of the slowest GPU)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
