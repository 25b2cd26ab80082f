"""Multi-process (one process per GPU, torchrun) data-parallel plumbing.

Each rank is one learner.  The batch sharding is the reference's
static_partition (engines/ssgd.py:16-25): rank r takes batches k*world + r of
the epoch pool, so a multi-process SSGD epoch consumes exactly the batches
the reference's SSGD learners would.  The gradient exchange uses
torch.distributed (NCCL on GPUs, gloo on CPU) — the comparison transport of
the north star; the single-process multi-device path uses the fused
canonical-order reduce kernel (ds_group_reduce) instead.
"""

from __future__ import annotations

import os

import numpy as np

from .schedule import epoch_minibatches, learning_rate, static_partition


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_batches(train_indices, batch_size: int, seed: int, epoch: int, rank: int, world: int) -> list:
    """This rank's minibatches of the epoch (static_partition of the pool)."""
    pool = epoch_minibatches(train_indices, batch_size, seed, epoch)
    if world == 1:
        return pool
    return static_partition(pool, world)[rank]


def allreduce_mean_(t, world: int, group=None) -> None:
    """In-place mean of a gradient tensor over the process group
    (engines/ssgd.py:85: allreduce / learners)."""
    import torch.distributed as dist

    if world > 1:
        dist.all_reduce(t, group=group)
        t.div_(world)


def ssgd_lr(schedule, epoch: int, k: int, q: int) -> float:
    """Learning rate of local iteration k of q (engines/ssgd.py:86)."""
    return learning_rate(schedule, epoch, k, q)


def shard_sizes(n_train: int, batch_size: int, world: int) -> list[int]:
    """Per-rank batch counts of one epoch (all equal: q = len(pool) // world)."""
    n_batches = -(-n_train // batch_size)
    return [n_batches // world] * world


__all__ = ["env_rank_world", "rank_batches", "allreduce_mean_", "ssgd_lr", "shard_sizes", "np"]
