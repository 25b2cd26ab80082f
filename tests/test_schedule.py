"""Host-side schedule layer: bit-exact
against the reference — live when /root/reference is importable, and always
against the committed golden vectors (tests/golden/schedule_golden.json,
produced by the reference via tests/golden/make_schedule_golden.py)."""

import json
import os

import numpy as np
import pytest

from paper_1904_04956_b200 import engines as E
from paper_1904_04956_b200 import schedule as S
from paper_1904_04956_b200.runtime import DelayModel, VirtualClock

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_golden.json")))


def test_epoch_minibatches_golden():
    for key, batches in GOLD["epoch_minibatches"].items():
        n, B, seed, ep = map(int, key.split("_"))
        mine = S.epoch_minibatches(np.arange(n), B, seed, ep)
        assert [b.tolist() for b in mine] == batches


def test_static_partition_golden():
    mine = S.static_partition(S.epoch_minibatches(np.arange(900), 160, 0, 1), 2)
    assert [[b.tolist() for b in p] for p in mine] == GOLD["static_partition_900_160_2"]
    # the short final batch lands on learner 2
    assert [len(b) for b in mine[1]] == [160, 160, 100]
    with pytest.raises(ValueError):
        S.static_partition([np.arange(3)], 2)


def test_learning_rate_golden():
    specs = {"large": S.large_batch_schedule(), "base": S.baseline_schedule(0.1)}
    for name, ep, k, n, lr in GOLD["learning_rate"]:
        assert S.learning_rate(specs[name], ep, k, n) == lr
    with pytest.raises(ValueError):
        S.learning_rate(specs["base"], 17)
    with pytest.raises(ValueError):
        S.learning_rate(specs["base"], 1, 5, 5)


def test_lr_known_answers():
    # tests/test_optim.py:19-57 of the reference: 0.1 start, 1.0 end of warm-up, anneal
    lb = S.large_batch_schedule()
    assert S.learning_rate(lb, 1, 0, 10) == pytest.approx(0.1)
    assert S.learning_rate(lb, 10, 9, 10) == pytest.approx(1.0)
    assert S.learning_rate(lb, 11, 0, 10) == pytest.approx(1.0 / np.sqrt(2))
    assert S.learning_rate(lb, 12, 0, 10) == pytest.approx(0.5)


def test_topology_golden():
    for lam, senders in GOLD["partners"].items():
        topo = S.Topology(int(lam))
        for i, partners in senders.items():
            assert [topo.partner(int(i), it) for it in range(1, 11)] == partners
    with pytest.raises(ValueError):
        S.Topology(3)
    with pytest.raises(ValueError):
        S.Topology(4).partner(2, 1)


def test_chunk_plans_golden():
    for key, bounds in GOLD["chunk_plans"].items():
        d, w, c = key.split("_")
        plan = S.make_chunk_plan(int(d), int(w), None if c == "None" else int(c))
        assert [list(b) for b in plan.bounds] == bounds
    assert S.allreduce_bytes_per_rank(100, 4, 8) == [2 * 3 * 25 * 8] * 4


def test_pool_exactly_once_threads():
    import threading

    for _ in range(50):
        pool = S.MinibatchPool([np.array([k]) for k in range(200)], 4)
        got = [[] for _ in range(4)]

        def worker(i):
            while True:
                d = pool.next(i + 1)
                if d is None:
                    return
                got[i].append(d[0])

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        allk = sorted(k for g in got for k in g)
        assert allk == list(range(200))
        assert sum(pool.counts) == 200


class _NullBackend:
    """Schedules are value-independent: replay them with
    no arithmetic at all."""

    elem_bytes = 8

    def __init__(self, dim):
        self.param_dim = dim

    def create(self, w0, momentum):
        return object()

    def __getattr__(self, name):
        if name in ("snapshot", "gradient", "sgd_step", "mix", "group_step", "group_average", "check", "sync"):
            return lambda *a, **k: None
        raise AttributeError(name)

    def average(self, members):
        return np.zeros(self.param_dim)

    def heldout_loss(self, w):
        return 0.0

    def weights(self, w):
        return np.zeros(self.param_dim)


class _Obj:
    kind = "quadratic"
    param_dim = 2
    regularization = 0.0


class _Data:
    def __init__(self, n):
        self.train_indices = np.arange(n - n // 10)
        self.heldout_indices = np.arange(n - n // 10, n)
        self.inputs = np.zeros((n, 2))


@pytest.mark.parametrize("lam", [2, 4, 8])
def test_adpsgd_schedule_golden(lam):
    g = GOLD["schedules"][f"adpsgd_{lam}"]
    res = E.run_adpsgd(_Obj(), _Data(600), S.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2,
                       batch_size=16, seed=3, delays=DelayModel(**{**GOLD["schedule_delays"], "slowdowns": {3: 2.0}}),
                       clock=VirtualClock(), record_trace=True, backend=_NullBackend(2))
    assert [r.minibatch_counts for r in res.records] == g["counts"]
    assert [r.epoch_wall_s for r in res.records] == g["wall"]
    assert [r.bytes_exchanged // 16 for r in res.records] == g["exchanges_bytes"]
    assert {str(k): v for k, v in res.trace["staleness_by_learner"].items()} == g["staleness_by_learner"]
    assert [list(p) for p in res.trace["exchanges"]] == g["pairs"]


@pytest.mark.parametrize("lam", [2, 4])
def test_ssgd_hybrid_schedule_golden(lam):
    d = DelayModel(**{**GOLD["schedule_delays"], "slowdowns": {3: 2.0}})
    res = E.run_ssgd(_Obj(), _Data(600), S.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2,
                     batch_size=16, seed=3, delays=d, clock=VirtualClock(), backend=_NullBackend(2))
    g = GOLD["schedules"][f"ssgd_{lam}"]
    assert [r.minibatch_counts for r in res.records] == g["counts"]
    assert [r.epoch_wall_s for r in res.records] == g["wall"]
    assert [r.bytes_exchanged // 8 for r in res.records] == g["bytes_per_elem"]
    d = DelayModel(**{**GOLD["schedule_delays"], "slowdowns": {3: 2.0}})
    res = E.run_hybrid(_Obj(), _Data(600), S.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2,
                       batch_size=16, seed=3, delays=d, clock=VirtualClock(), backend=_NullBackend(2))
    g = GOLD["schedules"][f"hybrid_{lam}"]
    assert [r.minibatch_counts for r in res.records] == g["counts"]
    assert [r.epoch_wall_s for r in res.records] == g["wall"]
    assert res.trace["staleness"].samples == g["staleness"]


def test_live_reference_schedule_functions(ref):
    data = ref.make_dataset("quadratic", 1000, 3, 0)
    for ep in (1, 2, 3):
        a = ref.epoch_minibatches(data, 37, 9, ep)
        b = S.epoch_minibatches(data, 37, 9, ep)
        assert all(np.array_equal(x, y) for x, y in zip(a, b)) and len(a) == len(b)
    from distsgd.engines.ssgd import static_partition

    a = static_partition(ref.epoch_minibatches(data, 37, 9, 1), 3)
    b = S.static_partition(S.epoch_minibatches(data, 37, 9, 1), 3)
    assert all(np.array_equal(x, y) for pa, pb in zip(a, b) for x, y in zip(pa, pb))
    for lam in (2, 6):
        t, u = ref.Topology(lam), S.Topology(lam)
        for i in range(1, lam + 1):
            assert t.left(i) == u.left(i) and t.right(i) == u.right(i) and t.role(i) == u.role(i)
