"""Host-side plan of the one-process-per-GPU strategies (each rank is one
learner; bench.py and p2p.PeerGroup execute it).

* Batch sharding: rank r takes batches k*world + r of the epoch pool — the
  reference's static_partition (engines/ssgd.py:16-25) — so a multi-process
  SSGD epoch consumes exactly the batches the reference's SSGD learners would.
* Per-iteration roles: `step_plan` says what rank r does at its k-th update
  under each strategy — who initiates an ADPSGD exchange and with whom
  (Topology, engines/common.py:38-75), which group an H-ADPSGD member
  synchronises with, whether its update must hold its own
  weight lock (the receiver's atomic region, engines/adpsgd.py:280-285).
"""

from __future__ import annotations

from dataclasses import dataclass

from .schedule import SENDER, Topology, epoch_minibatches, static_partition


def rank_batches(train_indices, batch_size: int, seed: int, epoch: int, rank: int, world: int) -> list:
    """This rank's minibatches of the epoch (static_partition of the pool)."""
    pool = epoch_minibatches(train_indices, batch_size, seed, epoch)
    if world == 1:
        return pool
    return static_partition(pool, world)[rank]


@dataclass(frozen=True)
class StepPlan:
    """What one rank does at one update.

    members     ranks of its synchronous group (SSGD: everyone; H-ADPSGD: its
                group; ADPSGD: itself)
    initiates   it starts a pairwise exchange after its update (a sender)
    partner     the rank it exchanges with this iteration (None: none)
    locked      its own update (or group step) holds its weight lock, because
                exchanges from other learners may land concurrently
    """

    members: tuple
    initiates: bool
    partner: int | None
    locked: bool


def step_plan(strategy: str, rank: int, world: int, k: int, groups: int = 2) -> StepPlan:
    """Plan of rank `rank` (0-based) at its k-th update (1-based iteration
    count, as Topology.partner uses it, engines/adpsgd.py:147-149)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside 0..{world - 1}")
    if k < 1:
        raise ValueError("iterations are 1-based")
    if strategy in ("single", "ssgd", "hybrid"):
        return StepPlan(tuple(range(world)), False, None, False)
    if strategy == "adpsgd":
        if world < 2 or world % 2:
            raise ValueError("adpsgd needs an even number of learners >= 2")
        topo = Topology(world)
        me = rank + 1
        if topo.role(me) == SENDER:
            return StepPlan((rank,), True, topo.partner(me, k) - 1, False)
        return StepPlan((rank,), False, None, True)
    if strategy == "hadpsgd":
        if groups < 2 or groups % 2 or world % groups:
            raise ValueError("hadpsgd needs an even group count dividing the learner count")
        size = world // groups
        gid, member = divmod(rank, size)
        topo = Topology(groups)
        mem = tuple(range(gid * size, (gid + 1) * size))
        if topo.role(gid + 1) == SENDER:
            return StepPlan(mem, True, (topo.partner(gid + 1, k) - 1) * size + member, False)
        return StepPlan(mem, False, None, True)
    raise ValueError(f"unknown strategy {strategy!r}")


def exchanges_at(strategy: str, world: int, k: int, groups: int = 2) -> list:
    """All (initiator, partner) pairs of iteration k (the edges in flight)."""
    out = []
    for r in range(world):
        p = step_plan(strategy, r, world, k, groups)
        if p.initiates:
            out.append((r, p.partner))
    return out


__all__ = ["rank_batches", "StepPlan", "step_plan", "exchanges_at"]
