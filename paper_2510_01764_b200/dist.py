"""Multi-GPU plumbing for the env step: one process per GPU,
contiguous global-id shards, one int64[4] all-reduce of episode statistics per
rollout, max-over-ranks timing.  Host logic only; backend-agnostic so the same
code runs over NCCL on GPUs and gloo in CPU tests."""
from __future__ import annotations

import os


def rank_info() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    g = lambda k, d: int(os.environ.get(k, d))
    return g("RANK", 0), g("WORLD_SIZE", 1), g("LOCAL_RANK", 0)


def shard(rank: int, world: int, n_per_rank: int) -> tuple[int, int]:
    """Global env ids owned by `rank`: [offset, offset + n_per_rank) (weak scaling)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * n_per_rank, n_per_rank


def shard_total(rank: int, world: int, total: int) -> tuple[int, int]:
    """Contiguous split of `total` global envs (strong scaling): sizes differ by at most 1."""
    base, rem = divmod(total, world)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def reduce_stats(stats, group=None):
    """Sum the int64[4] {returns, episodes, env_steps, error_flags} over ranks.
    Integer sums are order independent, so totals are bit-identical for any N."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def max_over_ranks(t, group=None):
    """Max of a 1-element timing tensor over ranks (the slowest rank defines the step)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t
