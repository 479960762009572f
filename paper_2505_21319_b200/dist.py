"""Data-parallel plumbing for the efunc fit step: one process per GPU, points sharded
across ranks, parameters replicated, the R^3 x 13 gradient summed with one all-reduce.

Pure host logic (no kernels here): which batch a rank draws, the global batch size that scales the
loss (Eq. loss, is a mean over the GLOBAL batch), and the gradient all-reduce.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_seed(seed: int, rank: int, step: int = 0) -> int:
    """Seed of the batch rank `rank` draws at `step`: distinct per (rank, step)."""
    return seed + 1000 * rank + 1_000_003 * step


def global_batch(points_per_rank: int, world_size: int) -> int:
    """J_global: every rank divides its loss and upstream by this, so the all-reduced gradient is
    the full-batch gradient (additivity over query subsets)."""
    return points_per_rank * world_size


def allreduce_grad(grad, group=None):
    """Sum the gradient over ranks in place (NCCL on GPU tensors, gloo on CPU tensors)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad
