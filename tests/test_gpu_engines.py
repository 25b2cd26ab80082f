"""Strategy-level parity on the GPU: the same engine code and the same
VirtualClock schedule drive (a) the device learners (GpuBackend, libds) and
(b) the float64 CPU oracle (oracle/blstm_ref.py through
tests/numpy_backend.py, whose engine is bit-identical to the reference
engines — tests/test_engines_cpu.py).  Integer streams (counts, staleness,
exchanges, virtual wall time) must be identical; weights after N steps agree
within the stated BF16-operand tolerance:
    ||(w_gpu - w0) - (w_ref - w0)|| / ||w_ref - w0|| <= 3e-2.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from numpy_backend import NumpyBackend  # noqa: E402
from oracle import blstm_ref as O  # noqa: E402
from paper_1904_04956_b200 import engines as E  # noqa: E402
from paper_1904_04956_b200.backend import GpuBackend  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective  # noqa: E402
from paper_1904_04956_b200.objective import make_blstm_dataset  # noqa: E402
from paper_1904_04956_b200.runtime import DelayModel, VirtualClock  # noqa: E402
from paper_1904_04956_b200.schedule import baseline_schedule  # noqa: E402

OBJ = BlstmObjective(layers=1, bottleneck=64, classes=256, frames=3)
SPEC = O.BlstmSpec(layers=1, input_dim=260, hidden=512, bottleneck=64, classes=256, frames=3)
DATA = make_blstm_dataset(OBJ, 90, seed=1)
XB = torch.from_numpy(DATA.inputs).bfloat16().double().numpy()  # the device sees bf16 features


def _oracle_grad(obj, w, batch, data):
    return O.loss_and_grad(SPEC, w, XB[batch], data.targets[batch])[1]


def _oracle_heldout(obj, w, data):
    idx = data.heldout_indices
    return O.loss(SPEC, w, XB[idx], data.targets[idx])


def _delays():
    return DelayModel(base_compute_s=2e-3, compute_jitter_s=1e-3, comm_latency_s=2e-4, comm_jitter_s=1e-4,
                      slowdowns={2: 1.7}, jitter_seed=3)


def _compare(run, **kw):
    w0 = O.initial_weights(SPEC, 4)
    sched = baseline_schedule(0.05, total_epochs=2)
    ref = run(OBJ, DATA, sched, seed=4, init_weights=w0, delays=_delays(), clock=VirtualClock(),
              backend=NumpyBackend(OBJ, DATA, _oracle_grad, _oracle_heldout), **kw)
    be = GpuBackend(OBJ, DATA, max_batch=16)
    gpu = run(OBJ, DATA, sched, seed=4, init_weights=w0, delays=_delays(), clock=VirtualClock(), backend=be, **kw)
    be.close()
    for a, b in zip(ref.records, gpu.records):
        assert a.minibatch_counts == b.minibatch_counts
        assert a.staleness_mean == b.staleness_mean and a.staleness_max == b.staleness_max
        assert a.epoch_wall_s == b.epoch_wall_s
        assert b.bytes_exchanged * 2 == a.bytes_exchanged  # 4 B/param on the device vs 8 B/param float64
        assert abs(a.heldout_loss - b.heldout_loss) <= 1e-2 * abs(a.heldout_loss)
    d_ref = ref.weights - w0
    d_gpu = gpu.weights - w0
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    print(run.__name__, "update rel err", rel)
    assert rel <= 3e-2
    return ref, gpu


def test_single_gpu_vs_oracle():
    _compare(E.run_single, epochs=1, batch_size=16)


def test_ssgd_gpu_vs_oracle():
    _compare(E.run_ssgd, learners=2, epochs=1, batch_size=8)


def test_adpsgd_gpu_vs_oracle():
    ref, gpu = _compare(E.run_adpsgd, learners=4, epochs=2, batch_size=8)
    assert ref.trace["staleness_by_learner"] == gpu.trace["staleness_by_learner"]


def test_hadpsgd_gpu_vs_oracle():
    _compare(E.run_hadpsgd, groups=2, group_size=2, epochs=1, batch_size=4)


def test_hybrid_gpu_vs_oracle():
    _compare(E.run_hybrid, learners=2, epochs=1, batch_size=8)


def _gpu_run(run, be, **kw):
    w0 = O.initial_weights(SPEC, 4)
    sched = baseline_schedule(0.05, total_epochs=2)
    res = run(OBJ, DATA, sched, seed=4, init_weights=w0, delays=_delays(), clock=VirtualClock(), backend=be, **kw)
    be.close()
    return res


@pytest.mark.parametrize("run,kw", [(E.run_adpsgd, dict(learners=4, epochs=2, batch_size=8)),
                                    (E.run_ssgd, dict(learners=2, epochs=1, batch_size=8)),
                                    (E.run_hadpsgd, dict(groups=2, group_size=2, epochs=1, batch_size=4)),
                                    (E.run_hybrid, dict(learners=2, epochs=1, batch_size=8))])
def test_per_learner_streams_bit_identical(run, kw):
    """Learners on their own CUDA streams (and devices, when the box has
    several) with event-ordered dependencies replay the schedule
    bit-identically to the single-stream layout."""
    ref = _gpu_run(run, GpuBackend(OBJ, DATA, max_batch=16), **kw)
    layouts = [dict(streams="per_learner")]
    if torch.cuda.device_count() >= 2:
        layouts.append(dict(devices=list(range(min(4, torch.cuda.device_count())))))
    for lay in layouts:
        got = _gpu_run(run, GpuBackend(OBJ, DATA, max_batch=16, **lay), **kw)
        assert np.array_equal(ref.weights, got.weights), lay
        for a, b in zip(ref.records, got.records):
            assert a == b, lay


def test_adpsgd_device_checksums():
    """checksum=True: every exchange validated with the device digest
    (ds_digest); results unchanged."""
    ref = _gpu_run(E.run_adpsgd, GpuBackend(OBJ, DATA, max_batch=16), learners=4, epochs=1, batch_size=8)
    got = _gpu_run(E.run_adpsgd, GpuBackend(OBJ, DATA, max_batch=16, streams="per_learner"), learners=4, epochs=1,
                   batch_size=8, checksum=True)
    assert np.array_equal(ref.weights, got.weights)
