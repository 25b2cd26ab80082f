"""Host-side schedule layer: everything that decides WHICH data and WHICH
weights each GPU operation sees.  These are integer / scalar computations
that must match the reference bit-exactly, so they
are restated here in plain Python/numpy and checked against the reference
by tests/test_schedule.py (and against committed golden vectors on the GPU
box, where the reference is absent).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# learning-rate schedules (optim.py:16-89)

@dataclass(frozen=True)
class LrSchedule:
    base_lr: float
    peak_lr: float
    warmup_epochs: int
    anneal_factor: float
    anneal_start_epoch: int
    total_epochs: int

    def __post_init__(self):
        checks = [
            (self.base_lr > 0, f"base_lr must be > 0, got {self.base_lr}"),
            (self.peak_lr >= self.base_lr, f"peak_lr ({self.peak_lr}) must be >= base_lr ({self.base_lr})"),
            (self.warmup_epochs >= 0, f"warmup_epochs must be >= 0, got {self.warmup_epochs}"),
            (0.0 < self.anneal_factor < 1.0, f"anneal_factor must lie in (0, 1), got {self.anneal_factor}"),
            (self.anneal_start_epoch > self.warmup_epochs,
             f"anneal_start_epoch ({self.anneal_start_epoch}) must be > warmup_epochs ({self.warmup_epochs})"),
            (self.total_epochs >= 1, f"total_epochs must be >= 1, got {self.total_epochs}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


_INV_SQRT2 = 1.0 / np.sqrt(2.0)


def large_batch_schedule(total_epochs: int = 16) -> LrSchedule:
    """0.1 -> 1.0 linear warm-up over 10 epochs, x 1/sqrt(2) per epoch from
    epoch 11 (optim.py:43-53)."""
    return LrSchedule(0.1, 1.0, 10, _INV_SQRT2, 11, total_epochs)


def baseline_schedule(lr: float = 0.1, total_epochs: int = 16) -> LrSchedule:
    """Constant lr, x 1/sqrt(2) per epoch from epoch 11 (optim.py:56-65)."""
    return LrSchedule(lr, lr, 0, _INV_SQRT2, 11, total_epochs)


def learning_rate(spec: LrSchedule, epoch: int, iter_in_epoch: int = 0, iters_per_epoch: int = 1) -> float:
    """optim.py:68-89: per-iteration warm-up interpolation, hold, per-epoch anneal."""
    if epoch < 1 or epoch > spec.total_epochs:
        raise ValueError(f"epoch {epoch} outside schedule range 1..{spec.total_epochs}")
    if iters_per_epoch < 1:
        raise ValueError(f"iters_per_epoch must be >= 1, got {iters_per_epoch}")
    if iter_in_epoch < 0 or iter_in_epoch >= iters_per_epoch:
        raise ValueError(f"iter_in_epoch {iter_in_epoch} outside 0..{iters_per_epoch - 1}")
    if epoch <= spec.warmup_epochs:
        span = spec.warmup_epochs * iters_per_epoch
        if span <= 1:
            return spec.peak_lr
        frac = ((epoch - 1) * iters_per_epoch + iter_in_epoch) / (span - 1)
        return spec.base_lr * (1.0 - frac) + spec.peak_lr * frac
    if epoch >= spec.anneal_start_epoch:
        return spec.peak_lr * spec.anneal_factor ** (epoch - spec.anneal_start_epoch + 1)
    return spec.peak_lr


# ---------------------------------------------------------------------------
# minibatch pools and sharding

def epoch_minibatches(train_indices: np.ndarray, batch_size: int, seed: int, epoch: int) -> list[np.ndarray]:
    """objectives.py:175-183: default_rng((seed, epoch)).shuffle of the
    training indices, cut into consecutive batch_size slices (last may be
    short).  Takes the index array (or a Dataset-like with .train_indices)."""
    if batch_size < 1:
        raise ValueError(f"batch_size must be >= 1, got {batch_size}")
    idx = getattr(train_indices, "train_indices", train_indices)
    order = np.array(idx, copy=True)
    np.random.default_rng((seed, epoch)).shuffle(order)
    return [order[s:s + batch_size] for s in range(0, len(order), batch_size)]


def static_partition(batches: list, learners: int) -> list[list]:
    """engines/ssgd.py:16-25: learner i (0-based) takes batches k*lambda + i,
    k < q = len // lambda (remainder dropped so collectives stay lockstep)."""
    q = len(batches) // learners
    if q == 0:
        raise ValueError(f"epoch pool of {len(batches)} minibatches cannot feed {learners} learners")
    return [batches[i:q * learners:learners] for i in range(learners)]


class MinibatchPool:
    """pool.py:16-46: lock-protected exactly-once hand-out of (position, batch)."""

    def __init__(self, batches: list, n_learners: int):
        self._mu = threading.Lock()
        self.n_learners = n_learners
        self.reset(batches)

    def reset(self, batches: list) -> None:
        with self._mu:
            self._items = list(batches)
            self._cursor = 0
            self.counts = [0] * self.n_learners

    @property
    def size(self) -> int:
        return len(self._items)

    def next(self, learner_id: int):
        with self._mu:
            k = self._cursor
            if k >= len(self._items):
                return None
            self._cursor = k + 1
            self.counts[learner_id - 1] += 1
            return k, self._items[k]


# ---------------------------------------------------------------------------
# ring topology (engines/common.py:38-75)

SENDER, RECEIVER = "sender", "receiver"


@dataclass(frozen=True)
class Topology:
    n_learners: int

    def __post_init__(self):
        if self.n_learners < 2 or self.n_learners % 2:
            raise ValueError(f"ring topology needs an even learner count >= 2, got {self.n_learners}")

    def role(self, learner_id: int) -> str:
        return SENDER if learner_id % 2 else RECEIVER

    def left(self, learner_id: int) -> int:
        return (learner_id - 2) % self.n_learners + 1

    def right(self, learner_id: int) -> int:
        return learner_id % self.n_learners + 1

    def partner(self, sender_id: int, iteration: int) -> int:
        if self.role(sender_id) != SENDER:
            raise ValueError(f"learner {sender_id} is not a sender")
        return self.right(sender_id) if iteration % 2 else self.left(sender_id)

    def senders(self) -> list[int]:
        return [i for i in range(1, self.n_learners + 1) if i % 2]

    def receivers(self) -> list[int]:
        return [i for i in range(1, self.n_learners + 1) if not i % 2]


# ---------------------------------------------------------------------------
# allreduce chunk plan (collective.py:22-57, 60-65)

@dataclass(frozen=True)
class ChunkPlan:
    world: int
    dim: int
    bounds: tuple

    @property
    def chunk_count(self) -> int:
        return len(self.bounds)

    def owner(self, chunk: int) -> int:
        return chunk % self.world

    def chunks_of(self, rank: int) -> list[int]:
        return list(range(rank, self.chunk_count, self.world))


def make_chunk_plan(dim: int, world: int, chunk_count: int | None = None) -> ChunkPlan:
    if world < 2:
        raise ValueError(f"ring allreduce needs at least 2 participants, got {world}")
    if dim < 1:
        raise ValueError(f"vector dim must be >= 1, got {dim}")
    c = world if chunk_count is None else chunk_count
    if c < world:
        raise ValueError(f"chunk_count ({c}) must be >= world ({world})")
    size = (dim + c - 1) // c
    return ChunkPlan(world, dim, tuple((min(j * size, dim), min(j * size + size, dim)) for j in range(c)))


def transfer_phase_count(world: int) -> int:
    if world < 2:
        raise ValueError(f"ring allreduce needs at least 2 participants, got {world}")
    return 2 * (world - 1)


def allreduce_bytes_per_rank(dim: int, world: int, elem_bytes: int = 4, chunk_count: int | None = None) -> list[int]:
    """Payload bytes each rank sends in one ring allreduce (collective.py:108-110):
    2(world-1) phases, each moving the chunks owned by the rank's send owner."""
    plan = make_chunk_plan(dim, world, chunk_count)
    sizes = [hi - lo for lo, hi in plan.bounds]
    out = []
    for r in range(world):
        tot = 0
        for s in range(world - 1):
            tot += sum(sizes[j] for j in plan.chunks_of((r - s) % world))
        for s in range(world - 1):
            tot += sum(sizes[j] for j in plan.chunks_of((r + 1 - s) % world))
        out.append(tot * elem_bytes)
    return out
