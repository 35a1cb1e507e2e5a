"""Multi-GPU sharding of independent sequences.

Frames within a sequence are sequential through the Kalman state and the
SGM recursion is sequential along each path, so the only parallelism across
GPUs is over independent sequences: each rank (one process per GPU) owns a
disjoint set of sequences and runs them as one batched context.  There is
no data-path collective; ranks meet only at the timing barrier and the
max-over-ranks reduction of the elapsed time.
"""

from __future__ import annotations

__all__ = ["rank_sequences", "max_over_ranks", "barrier", "world"]


def world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    import os
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def rank_sequences(rank: int, world_size: int, per_rank: int, seed0: int = 1000):
    """Disjoint sequence seeds of one rank (weak scaling: per_rank fixed)."""
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} outside world of {world_size}")
    base = seed0 + rank * per_rank
    return list(range(base, base + per_rank))


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
