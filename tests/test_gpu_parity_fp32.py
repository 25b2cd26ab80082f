"""FP32-parity mode (DS_PREC_FP32: every GEMM on tcgen05 kind::tf32 with the
3xTF32 split, fp32 activations / cell state / soft-max) against the float64
CPU oracle (oracle/blstm_ref.py, objectives.py:236-263) and the
reference momentum step (optim.py:109-121).

Stated FP32-mode tolerances (BASELINE config 2 and smaller shapes):
  3xTF32 GEMM vs float64                      max |err| / max |C| <= 1.5e-5 (K <= 1000)
  loss                                        |rel| <= 1e-5
  gradient per tensor block                   rel L2 <= 1e-3, cosine >= 0.999999
  theta after 3 momentum steps (config 2)     update rel <= 1e-3
  engine replay (ADPSGD lambda=2 / SSGD)      update rel <= 1e-3, integer streams identical
(the BF16 perf mode's bounds are in tests/test_gpu_config2.py).
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import blstm_ref as O  # noqa: E402
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, offsets  # noqa: E402

REPORT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                      "parity_fp32.json")


def _save(key, val):
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    d = {}
    if os.path.exists(REPORT):
        with open(REPORT) as f:
            d = json.load(f)
    d[key] = val
    with open(REPORT, "w") as f:
        json.dump(d, f, indent=1)


def _blocks(obj, g, g_ref):
    out = {}
    for k, v in offsets(obj).items():
        if k == "total":
            continue
        o, shape = v
        n = int(np.prod(shape))
        a, r = g[o:o + n], g_ref[o:o + n]
        if np.linalg.norm(r) == 0:
            continue
        rel = float(np.linalg.norm(a - r) / np.linalg.norm(r))
        cos = float(a @ r / max(np.linalg.norm(a) * np.linalg.norm(r), 1e-30))
        out[str(k)] = (rel, cos)
    return out


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 200, 260), (5, 2048, 512), (777, 96, 1000)])
def test_gemm_tf32x3_matches_float64(M, N, K):
    lib = _lib.load()
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((N, K)).astype(np.float32)
    A, Bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    C = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    _lib.check(lib.ds_debug_gemm_tf32x3(A.data_ptr(), K, Bt.data_ptr(), K, C.data_ptr(), N, M, N, K, 0,
                                        _lib.stream_ptr()))
    torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(C.cpu().numpy() - ref).max() / np.abs(ref).max()
    print("gemm3", M, N, K, err)
    assert err <= 1.5e-5
    # accumulate: C += A B^T
    _lib.check(lib.ds_debug_gemm_tf32x3(A.data_ptr(), K, Bt.data_ptr(), K, C.data_ptr(), N, M, N, K, 1,
                                        _lib.stream_ptr()))
    torch.cuda.synchronize()
    err2 = np.abs(C.cpu().numpy() - 2 * ref).max() / np.abs(2 * ref).max()
    assert err2 <= 1.5e-5


@pytest.mark.parametrize("layers,B,T,classes,bott,din", [(2, 24, 6, 512, 256, 260), (1, 7, 3, 1008, 64, 40),
                                                          (1, 300, 2, 256, 128, 260), (3, 5, 1, 384, 256, 260)])
def test_fp32_mode_matches_oracle(layers, B, T, classes, bott, din):
    obj = BlstmObjective(layers=layers, classes=classes, frames=T, bottleneck=bott, input_dim=din)
    spec = O.BlstmSpec(layers=layers, input_dim=din, hidden=512, bottleneck=bott, classes=classes, frames=T)
    x, y, _, _ = O.make_dataset(spec, B + 3, seed=13)
    w = O.initial_weights(spec, 13)
    batch = np.random.default_rng(1).permutation(len(x))[:B]
    xb = torch.from_numpy(x).bfloat16().double().numpy()
    loss_ref, g_ref = O.loss_and_grad(spec, w, xb[batch], y[batch])
    L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=w, precision="fp32")
    L.gradient(batch)
    L.check_finite()
    loss = L.mean_loss()
    g = L.grad.double().cpu().numpy()
    rel_loss = abs(loss - loss_ref) / abs(loss_ref)
    blocks = _blocks(obj, g, g_ref)
    worst = max(blocks.values())
    print("fp32 mode", (layers, B, T, classes), "loss rel", rel_loss, "worst block", worst)
    assert rel_loss <= 1e-5
    for k, (rel, cos) in blocks.items():
        assert rel <= 1e-3 and cos >= 0.999999, (k, rel, cos)
    L.close()


def test_fp32_mode_config2_gradient_and_three_steps():
    """BASELINE config 2 itself (6 x 1024 BLSTM, T=21, 32000 classes, B=256):
    gradient at theta_0 and theta after 3 momentum steps vs float64."""
    obj, spec, B, mu, lrs = BlstmObjective(), O.BlstmSpec(), 256, 0.9, (0.1, 0.1, 0.1)
    x, y, _, _ = O.make_dataset(spec, 3 * B + 16, seed=21)
    xb = torch.from_numpy(x).bfloat16().double().numpy()
    w0 = O.initial_weights(spec, 21)
    perm = np.random.default_rng(5).permutation(len(x))
    batches = [perm[s * B:(s + 1) * B] for s in range(len(lrs))]
    w, v, ref_loss = w0.copy(), np.zeros_like(w0), []
    for s, lr in enumerate(lrs):
        loss, g = O.loss_and_grad(spec, w, xb[batches[s]], y[batches[s]])
        ref_loss.append(loss)
        if s == 0:
            g0 = g
        v = mu * v + g
        w = w - lr * v
    L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=w0, momentum=mu, precision="fp32")
    gpu_loss = []
    for s, lr in enumerate(lrs):
        L.train_step(batches[s], lr)
        L.check_finite()
        gpu_loss.append(L.mean_loss())
        if s == 0:
            gg0 = L.grad.double().cpu().numpy()
    w_gpu = L.weights()
    L.close()
    blocks = _blocks(obj, gg0, g0)
    tot = float(np.linalg.norm(gg0 - g0) / np.linalg.norm(g0))
    upd = float(np.linalg.norm((w_gpu - w0) - (w - w0)) / np.linalg.norm(w - w0))
    loss_rel = [abs(a - b) / abs(b) for a, b in zip(gpu_loss, ref_loss)]
    print("fp32 config2: grad total rel", tot, "worst", max(blocks.values()), "update rel", upd, "loss rel", loss_rel)
    _save("fp32_config2", {"grad_rel_total": tot, "blocks": blocks, "theta3_update_rel": upd,
                           "loss_rel_per_step": loss_rel, "loss_gpu": gpu_loss, "loss_ref": ref_loss})
    assert max(loss_rel) <= 1e-5
    for k, (rel, cos) in blocks.items():
        assert rel <= 1e-3 and cos >= 0.999999, (k, rel, cos)
    assert upd <= 1e-3


@pytest.mark.parametrize("strategy", ["adpsgd", "ssgd"])
def test_fp32_mode_engine_replay_matches_oracle_engine(strategy):
    """The drop-in engines on FP32-mode device learners vs the same engine on
    float64 oracle learners (same VirtualClock schedule)."""
    from numpy_backend import NumpyBackend

    from paper_1904_04956_b200 import engines as E
    from paper_1904_04956_b200.backend import GpuBackend
    from paper_1904_04956_b200.objective import make_blstm_dataset
    from paper_1904_04956_b200.runtime import DelayModel, VirtualClock
    from paper_1904_04956_b200.schedule import baseline_schedule

    obj = BlstmObjective(layers=2, bottleneck=64, classes=256, frames=5)
    spec = O.BlstmSpec(layers=2, input_dim=260, hidden=512, bottleneck=64, classes=256, frames=5)
    data = make_blstm_dataset(obj, 90, seed=1)
    xb = torch.from_numpy(data.inputs).bfloat16().double().numpy()

    def grad(o, w, batch, d):
        return O.loss_and_grad(spec, w, xb[batch], d.targets[batch])[1]

    def held(o, w, d):
        return O.loss(spec, w, xb[d.heldout_indices], d.targets[d.heldout_indices])

    def delays():
        return DelayModel(base_compute_s=2e-3, compute_jitter_s=1e-3, comm_latency_s=2e-4, comm_jitter_s=1e-4,
                          slowdowns={2: 1.7}, jitter_seed=3)

    w0 = O.initial_weights(spec, 4)
    sched = baseline_schedule(0.05, total_epochs=2)
    run = E.run_adpsgd if strategy == "adpsgd" else E.run_ssgd
    kw = dict(learners=2, epochs=2, batch_size=8, seed=4, init_weights=w0)
    ref = run(obj, data, sched, delays=delays(), clock=VirtualClock(), backend=NumpyBackend(obj, data, grad, held),
              **kw)
    be = GpuBackend(obj, data, max_batch=8, precision="fp32")
    gpu = run(obj, data, sched, delays=delays(), clock=VirtualClock(), backend=be, **kw)
    be.close()
    for a, b in zip(ref.records, gpu.records):
        assert a.minibatch_counts == b.minibatch_counts
        assert (a.staleness_mean, a.staleness_max, a.epoch_wall_s) == (b.staleness_mean, b.staleness_max,
                                                                       b.epoch_wall_s)
        assert abs(a.heldout_loss - b.heldout_loss) <= 1e-5 * abs(a.heldout_loss)
    rel = float(np.linalg.norm((gpu.weights - w0) - (ref.weights - w0)) / np.linalg.norm(ref.weights - w0))
    print(strategy, "fp32 engine update rel", rel)
    assert rel <= 1e-3
