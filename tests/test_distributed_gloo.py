"""The one-process-per-GPU host plan (paper_1904_04956_b200/distributed.py)
across a real world-4 process group (gloo on CPU): every rank computes its
own batches and per-iteration roles; gathered, they must form the
reference's schedule — SSGD shards disjoint and covering the truncated pool
(static_partition, engines/ssgd.py:16-25); ADPSGD exchanges a matching of
senders onto receivers with the Topology partners (engines/common.py:38-75),
receivers locked; H-ADPSGD groups partitioning the ranks with member r of
partner groups paired."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1904_04956_b200.distributed import rank_batches, step_plan

    mine = {"batches": [b.tolist() for b in rank_batches(np.arange(1000), 32, 3, 2, rank, world)],
            "adpsgd": [step_plan("adpsgd", rank, world, k) for k in range(1, 9)],
            "hadpsgd": [step_plan("hadpsgd", rank, world, k, groups=2) for k in range(1, 9)],
            "ssgd": step_plan("ssgd", rank, world, 1)}
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank == 0:
        out["plans"] = got
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_world_host_plan(world):
    from paper_1904_04956_b200.schedule import SENDER, Topology, epoch_minibatches

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    plans = out["plans"]
    # SSGD: shards disjoint, covering the pool truncated to q*world, in static_partition order
    pool = epoch_minibatches(np.arange(1000), 32, 3, 2)
    q = len(pool) // world
    for r in range(world):
        assert plans[r]["batches"] == [pool[k * world + r].tolist() for k in range(q)]
        assert plans[r]["ssgd"].members == tuple(range(world)) and not plans[r]["ssgd"].initiates
    # ADPSGD: senders (odd ids) initiate to their Topology partner; receivers locked; a matching per step
    topo = Topology(world)
    for k in range(8):
        edges = [(r, plans[r]["adpsgd"][k].partner) for r in range(world) if plans[r]["adpsgd"][k].initiates]
        assert [r + 1 for r, _ in edges] == topo.senders()
        assert all(p + 1 == topo.partner(r + 1, k + 1) for r, p in edges)
        assert len({p for _, p in edges}) == len(edges)  # each receiver mixes with one sender at a time
        for r in range(world):
            assert plans[r]["adpsgd"][k].locked == (topo.role(r + 1) != SENDER)
    # H-ADPSGD (2 groups): groups partition the ranks; member r of the sender group pairs member r of the other
    size = world // 2
    for k in range(8):
        groups = {plans[r]["hadpsgd"][k].members for r in range(world)}
        assert sorted(x for g in groups for x in g) == list(range(world)) and len(groups) == 2
        for r in range(world):
            p = plans[r]["hadpsgd"][k]
            if p.initiates:
                assert r < size and p.partner == size + r and not p.locked
            else:
                assert r >= size and p.locked and p.partner is None
