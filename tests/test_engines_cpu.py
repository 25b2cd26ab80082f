"""Engine + runtime restatement vs the reference engines, on CPU.

The engines of paper_1904_04956_b200/engines.py drive a float64 numpy backend
(tests/numpy_backend.py) that performs the reference's own arithmetic; under
the same VirtualClock delays the results must be bit-identical to the
reference engines: final weights, per-epoch records (held-out loss, virtual
wall time, minibatch counts, staleness, bytes) and staleness samples.  This
pins the schedule (draw order, partners, update/mix interleaving) that the
GPU runs replay.
"""

import numpy as np
import pytest

from numpy_backend import NumpyBackend
from paper_1904_04956_b200 import engines as E
from paper_1904_04956_b200.runtime import DelayModel, VirtualClock

FIELDS = ("epoch", "heldout_loss", "epoch_wall_s", "minibatch_counts", "staleness_mean", "staleness_max",
          "bytes_exchanged")


def _problem(ref, kind, n=400, dim=6, seed=3):
    obj = ref.make_objective(kind, dim)
    data = ref.make_dataset(kind, n, dim, seed)
    return obj, data


def _backend(ref, obj, data):
    import distsgd.objectives as ro

    return NumpyBackend(obj, data, ro.gradient, ro.heldout_loss)


def _delays(ref_mod, jitter=True, straggler=None):
    kw = dict(base_compute_s=2e-3, compute_jitter_s=1e-3 if jitter else 0.0, comm_latency_s=2e-4,
              comm_jitter_s=1e-4 if jitter else 0.0, jitter_seed=11)
    if straggler:
        kw["slowdowns"] = straggler
    return ref_mod.DelayModel(**kw), DelayModel(**kw)


def _same_records(a, b):
    assert len(a) == len(b)
    for ra, rb in zip(a, b):
        for f in FIELDS:
            assert getattr(ra, f) == getattr(rb, f), (f, getattr(ra, f), getattr(rb, f))


@pytest.mark.parametrize("kind", ["logistic", "tiny-mlp"])
def test_single_bit_identical(ref, kind):
    obj, data = _problem(ref, kind)
    sched = ref.baseline_schedule(0.1, total_epochs=3)
    rd, md = _delays(ref)
    r = ref.run_single(obj, data, sched, epochs=2, batch_size=32, seed=5, delays=rd, clock=ref.VirtualClock())
    m = E.run_single(obj, data, sched, epochs=2, batch_size=32, seed=5, delays=md, clock=VirtualClock(),
                     backend=_backend(ref, obj, data))
    assert np.array_equal(r.weights, m.weights)
    _same_records(r.records, m.records)


@pytest.mark.parametrize("learners,chunks", [(2, None), (3, 5), (4, None)])
def test_ssgd_bit_identical(ref, learners, chunks):
    obj, data = _problem(ref, "logistic")
    sched = ref.large_batch_schedule(total_epochs=16)
    rd, md = _delays(ref, straggler={2: 1.5})
    r = ref.run_ssgd(obj, data, sched, learners=learners, epochs=2, batch_size=20, seed=1, delays=rd,
                     clock=ref.VirtualClock(), chunk_count=chunks)
    m = E.run_ssgd(obj, data, sched, learners=learners, epochs=2, batch_size=20, seed=1, delays=md,
                   clock=VirtualClock(), chunk_count=chunks, backend=_backend(ref, obj, data))
    assert np.array_equal(r.weights, m.weights)
    _same_records(r.records, m.records)


@pytest.mark.parametrize("learners", [2, 4, 8])
@pytest.mark.parametrize("kind", ["logistic", "tiny-mlp"])
def test_adpsgd_bit_identical(ref, learners, kind):
    obj, data = _problem(ref, kind)
    sched = ref.baseline_schedule(0.05, total_epochs=4)
    rd, md = _delays(ref, straggler={3: 2.0} if learners > 2 else None)
    r = ref.run_adpsgd(obj, data, sched, learners=learners, epochs=2, batch_size=16, seed=2, delays=rd,
                       clock=ref.VirtualClock())
    m = E.run_adpsgd(obj, data, sched, learners=learners, epochs=2, batch_size=16, seed=2, delays=md,
                     clock=VirtualClock(), backend=_backend(ref, obj, data))
    assert np.array_equal(r.weights, m.weights)
    _same_records(r.records, m.records)
    assert r.trace["staleness"].samples == m.trace["staleness"].samples
    assert r.trace["staleness_by_learner"] == m.trace["staleness_by_learner"]


def test_adpsgd_zero_delay_schedule(ref):
    """Zero delay starves senders in the reference: same here."""
    obj, data = _problem(ref, "quadratic")
    sched = ref.baseline_schedule(0.05, total_epochs=2)
    r = ref.run_adpsgd(obj, data, sched, learners=4, epochs=1, batch_size=16, seed=0, clock=ref.VirtualClock())
    m = E.run_adpsgd(obj, data, sched, learners=4, epochs=1, batch_size=16, seed=0, clock=VirtualClock(),
                     backend=_backend(ref, obj, data))
    assert np.array_equal(r.weights, m.weights)
    _same_records(r.records, m.records)


@pytest.mark.parametrize("learners", [2, 4])
def test_hybrid_bit_identical(ref, learners):
    obj, data = _problem(ref, "tiny-mlp")
    sched = ref.baseline_schedule(0.05, total_epochs=3)
    rd, md = _delays(ref)
    r = ref.run_hybrid(obj, data, sched, learners=learners, epochs=2, batch_size=16, seed=4, delays=rd,
                       clock=ref.VirtualClock())
    m = E.run_hybrid(obj, data, sched, learners=learners, epochs=2, batch_size=16, seed=4, delays=md,
                     clock=VirtualClock(), backend=_backend(ref, obj, data))
    assert np.array_equal(r.weights, m.weights)
    _same_records(r.records, m.records)
    assert r.trace["staleness"].samples == m.trace["staleness"].samples


def test_hadpsgd_matches_adpsgd_of_groups(ref):
    """H-ADPSGD (G groups x g members, m per member) == reference ADPSGD with
    G learners and batch g*m: identical schedule; weights equal up to the
    float64 regrouping of the per-slice gradient sum."""
    obj, data = _problem(ref, "logistic", n=500)
    sched = ref.baseline_schedule(0.05, total_epochs=3)
    rd, md = _delays(ref)
    r = ref.run_adpsgd(obj, data, sched, learners=2, epochs=2, batch_size=40, seed=6, delays=rd,
                       clock=ref.VirtualClock())
    m = E.run_hadpsgd(obj, data, sched, groups=2, group_size=4, epochs=2, batch_size=10, seed=6, delays=md,
                      clock=VirtualClock(), backend=_backend(ref, obj, data))
    np.testing.assert_allclose(m.weights, r.weights, rtol=1e-12, atol=1e-13)
    for ra, rb in zip(r.records, m.records):
        assert ra.minibatch_counts == rb.minibatch_counts
        assert ra.staleness_mean == rb.staleness_mean and ra.staleness_max == rb.staleness_max
        assert ra.epoch_wall_s == rb.epoch_wall_s
        assert rb.bytes_exchanged == 4 * ra.bytes_exchanged  # four member payloads per exchange
    assert r.trace["staleness"].samples == m.trace["staleness"].samples


def test_engine_failure_epoch(ref):
    obj, data = _problem(ref, "logistic")
    sched = ref.baseline_schedule(0.1, total_epochs=3)
    w = np.full(obj.param_dim, np.nan)
    with pytest.raises(E.EngineFailure) as ei:
        E.run_single(obj, data, sched, epochs=1, batch_size=32, seed=0, init_weights=w,
                     backend=_backend(ref, obj, data))
    assert ei.value.epoch == 1


def test_validation_errors(ref):
    obj, data = _problem(ref, "logistic")
    sched = ref.baseline_schedule(0.1, total_epochs=2)
    be = _backend(ref, obj, data)
    with pytest.raises(ValueError):
        E.run_adpsgd(obj, data, sched, learners=3, epochs=1, batch_size=8, seed=0, backend=be)
    with pytest.raises(ValueError):
        E.run_ssgd(obj, data, sched, learners=1, epochs=1, batch_size=8, seed=0, backend=be)
    with pytest.raises(ValueError):
        E.run_single(obj, data, sched, epochs=5, batch_size=8, seed=0, backend=be)


def test_adpsgd_checksum_mode(ref):
    """Debug payload checksums (WeightMessage, common.py:78-104): identical
    results with checksums on, and a mix that leaves the two learners with
    different weights is caught as ChecksumError."""
    obj, data = _problem(ref, "logistic")
    sched = ref.baseline_schedule(0.1, total_epochs=2)
    _, md = _delays(ref)
    kw = dict(learners=4, epochs=2, batch_size=16, seed=2, clock=VirtualClock())
    a = E.run_adpsgd(obj, data, sched, delays=md, backend=_backend(ref, obj, data), **kw)
    _, md2 = _delays(ref)
    kw["clock"] = VirtualClock()
    b = E.run_adpsgd(obj, data, sched, delays=md2, backend=_backend(ref, obj, data), checksum=True, **kw)
    assert np.array_equal(a.weights, b.weights)
    _same_records(a.records, b.records)

    class Torn(NumpyBackend):
        def mix(self, x, y):
            super().mix(x, y)
            y.w = y.w + 1e-12  # the two sides no longer hold the identical mean

    _, md3 = _delays(ref)
    kw["clock"] = VirtualClock()
    with pytest.raises(E.ChecksumError):
        import distsgd.objectives as ro

        E.run_adpsgd(obj, data, sched, delays=md3, backend=Torn(obj, data, ro.gradient, ro.heldout_loss),
                     checksum=True, **kw)
