"""The clocks of paper_1904_04956_b200/runtime.py on their own: ordering
contract, deadlock detection, failure propagation, RealClock engine runs
(throughput mode) and DelayModel streams equal to the reference's."""

import threading

import numpy as np
import pytest

from numpy_backend import NumpyBackend
from paper_1904_04956_b200 import engines as E
from paper_1904_04956_b200.runtime import (DeadlockError, DelayModel, RealClock, RunAborted, VirtualClock,
                                           make_clock)


def test_virtual_order_is_time_then_sequence():
    clk = VirtualClock()
    log = []
    ch = clk.channel(lambda: 0.5)

    def a():
        clk.sleep(1.0)
        log.append(("a", clk.now()))
        ch.put("x")
        ch.put("y")

    def b():
        log.append(("b0", clk.now()))
        log.append((ch.get(), clk.now()))
        log.append((ch.get(), clk.now()))

    def c():
        clk.sleep(1.0)  # same time as a, later sequence number
        log.append(("c", clk.now()))

    clk.run([a, b, c])
    assert log == [("b0", 0.0), ("a", 1.0), ("c", 1.0), ("x", 1.5), ("y", 1.5)]


def test_channel_deliveries_never_overtake():
    clk = VirtualClock()
    delays = iter([1.0, 0.1])
    ch = clk.channel(lambda: next(delays))
    got = []

    def prod():
        ch.put(1)
        ch.put(2)  # shorter latency, still delivered after 1 (link FIFO)

    def cons():
        got.append((ch.get(), clk.now()))
        got.append((ch.get(), clk.now()))

    clk.run([prod, cons])
    assert got == [(1, 1.0), (2, 1.0)]


def test_deadlock_detected_and_reported():
    clk = VirtualClock()
    a_ch, b_ch = clk.channel(), clk.channel()
    with pytest.raises(DeadlockError, match="actor-0"):
        clk.run([lambda: a_ch.get(), lambda: b_ch.get()])


def test_actor_failure_tears_down_the_run():
    clk = VirtualClock()
    ch = clk.channel()
    reached = []

    def bad():
        clk.sleep(0.1)
        raise KeyError("boom")

    def blocked():
        try:
            ch.get()
        except RunAborted:
            reached.append(True)
            raise

    with pytest.raises(KeyError):
        clk.run([bad, blocked])
    assert reached == [True]


def test_single_use_and_outside_actor():
    clk = VirtualClock()
    clk.run([lambda: None])
    with pytest.raises(RuntimeError):
        clk.run([lambda: None])
    with pytest.raises(RuntimeError):
        VirtualClock().sleep(1.0)


def test_real_clock_latency_and_abort():
    clk = make_clock("real")
    ch = clk.channel(lambda: 0.05)
    out = []

    def prod():
        ch.put(clk.now())

    def cons():
        t_sent = ch.get()
        out.append(clk.now() - t_sent)

    clk.run([prod, cons])
    assert out and out[0] >= 0.045
    clk2 = RealClock()
    ch2 = clk2.channel()

    def waiter():
        ch2.get()

    def fail():
        raise ValueError("x")

    with pytest.raises(ValueError):
        clk2.run([waiter, fail])


def test_delay_model_streams_match_reference(ref):
    kw = dict(base_compute_s=2e-3, compute_jitter_s=1e-3, comm_latency_s=2e-4, comm_jitter_s=1e-4,
              slowdowns={3: 2.5}, stagger_s=0.01, jitter_seed=7)
    mine, theirs = DelayModel(**kw), ref.DelayModel(**kw)
    for learner in (1, 3):
        f, g = mine.compute_delay_fn(learner), theirs.compute_delay_fn(learner)
        assert [f() for _ in range(20)] == [g() for _ in range(20)]
        assert mine.initial_stagger(learner) == theirs.initial_stagger(learner)
    f, g = mine.comm_delay_fn(4), theirs.comm_delay_fn(4)
    assert [f() for _ in range(20)] == [g() for _ in range(20)]
    assert DelayModel().comm_delay_fn(1) is None and ref.DelayModel().comm_delay_fn(1) is None
    with pytest.raises(ValueError):
        DelayModel(slowdowns={2: 0.5})


def test_adpsgd_on_real_clock_conserves_pairs(ref):
    """Throughput mode: free-running actor threads.  Schedules are not
    reproducible, but every sender update is followed by exactly one
    exchange, and the pair mixes conserve the learners' sum (adpsgd_mix,
    engines/adpsgd.py:36-43; tests/test_adpsgd.py:84-94 of the reference)."""
    import distsgd.objectives as ro

    obj = ref.make_objective("logistic", 6)
    data = ref.make_dataset("logistic", 400, 6, 3)
    be = NumpyBackend(obj, data, ro.gradient, ro.heldout_loss)
    sched = ref.baseline_schedule(0.1, total_epochs=2)
    res = E.run_adpsgd(obj, data, sched, learners=4, epochs=2, batch_size=16, seed=1, clock=RealClock(),
                       delays=DelayModel(base_compute_s=1e-3, comm_latency_s=2e-4), backend=be, record_trace=True)
    assert np.all(np.isfinite(res.weights))
    assert sum(res.records[-1].minibatch_counts) == len(ref.epoch_minibatches(data, 16, 1, 2))
    n_updates_senders = sum(1 for i in (1, 3) for _ in res.trace["staleness_by_learner"][i])
    assert len(res.trace["exchanges"]) == n_updates_senders
    assert threading.active_count() < 50
