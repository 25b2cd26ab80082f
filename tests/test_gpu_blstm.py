"""End-to-end parity of the GPU BLSTM training step against the float64 CPU
oracle (oracle/blstm_ref.py) on identical inputs, plus the sync kernels
against float32 restatements of the reference arithmetic.

Stated tolerances (BF16 tensor-core operands, FP32 accumulation/state):
  loss                      : |rel| <= 5e-3
  gradient, per tensor block: ||g - g_ref|| / ||g_ref|| <= 2.5e-2 and cosine >= 0.9995
  sgd_step / adpsgd_mix / canonical allreduce : bit-exact vs float32 numpy
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import blstm_ref as O  # noqa: E402
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, offsets  # noqa: E402


def _spec(obj):
    return O.BlstmSpec(layers=obj.layers, input_dim=obj.input_dim, hidden=512, bottleneck=obj.bottleneck,
                       classes=obj.classes, frames=obj.frames)


@pytest.mark.parametrize("layers,B,T,classes", [(2, 24, 6, 512), (1, 136, 5, 256), (1, 40, 3, 1280), (1, 8, 3, 32000),
                                                  (1, 24, 4, 1008)])  # 1008: not a multiple of 128 -> GEMM-epilogue path
def test_fwd_bwd_matches_oracle(layers, B, T, classes):
    obj = BlstmObjective(layers=layers, classes=classes, frames=T)
    spec = _spec(obj)
    assert spec.param_dim == obj.param_dim
    x, y, _, _ = O.make_dataset(spec, 2 * B + 3, seed=5)
    w = O.initial_weights(spec, 5)
    rng = np.random.default_rng(0)
    batch = rng.permutation(len(x))[:B]
    # the GPU consumes bf16 features: give the oracle the same rounded inputs
    xb = torch.from_numpy(x).bfloat16().double().numpy()
    loss_ref, g_ref = O.loss_and_grad(spec, w, xb[batch], y[batch])

    L = Learner(obj, DeviceDataset(x, y), max_batch=2 * B, theta0=w)
    L.gradient(batch)
    L.check_finite()
    loss = L.mean_loss()
    g = L.grad.double().cpu().numpy()
    assert abs(loss - loss_ref) <= 5e-3 * abs(loss_ref), (loss, loss_ref)
    report = {}
    for k, v in offsets(obj).items():
        if k == "total":
            continue
        o, shape = v
        n = int(np.prod(shape))
        a, r = g[o:o + n], g_ref[o:o + n]
        rel = np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-30)
        cos = float(a @ r / max(np.linalg.norm(a) * np.linalg.norm(r), 1e-30))
        report[k] = (rel, cos)
    print(report)
    for k, (rel, cos) in report.items():
        assert rel <= 2.5e-2 and cos >= 0.9995, (k, rel, cos)
    # second call reuses the cached CUDA graph and must give the same result
    L.gradient(batch)
    L.stream.synchronize()
    assert torch.equal(L.grad.double().cpu(), torch.from_numpy(g))
    L.close()


@pytest.mark.parametrize("classes", [1280, 1008])  # fused soft-max kernels / GEMM-epilogue path
def test_large_output_bias_matches_oracle(classes):
    """Output biases far from the initial 0.1 N(0,1) scale (N(0, 3), a few at +-20): the fused
    gradient kernel multiplies by exp(b) after the exponential and folds 1/frames into the
    exponent; both must stay within the stated tolerances against the float64 oracle."""
    B, T = 24, 4
    obj = BlstmObjective(layers=1, classes=classes, frames=T)
    spec = _spec(obj)
    x, y, _, _ = O.make_dataset(spec, 2 * B + 3, seed=9)
    w = O.initial_weights(spec, 9)
    o, shape = offsets(obj)["bo"]
    rng = np.random.default_rng(3)
    bo = 3.0 * rng.standard_normal(shape[0])
    bo[rng.choice(shape[0], 6, replace=False)] = [20.0, -20.0, 18.0, -18.0, 15.0, 12.0]
    w = w.copy()
    w[o:o + shape[0]] = bo
    batch = rng.permutation(len(x))[:B]
    xb = torch.from_numpy(x).bfloat16().double().numpy()
    loss_ref, g_ref = O.loss_and_grad(spec, w, xb[batch], y[batch])
    L = Learner(obj, DeviceDataset(x, y), max_batch=2 * B, theta0=w)
    L.gradient(batch)
    L.check_finite()
    loss = L.mean_loss()
    g = L.grad.double().cpu().numpy()
    assert abs(loss - loss_ref) <= 5e-3 * abs(loss_ref), (loss, loss_ref)
    for k, v in offsets(obj).items():
        if k == "total":
            continue
        oo, sh = v
        n = int(np.prod(sh))
        a, r = g[oo:oo + n], g_ref[oo:oo + n]
        rel = np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-30)
        cos = float(a @ r / max(np.linalg.norm(a) * np.linalg.norm(r), 1e-30))
        assert rel <= 2.5e-2 and cos >= 0.9995, (k, rel, cos)
    L.close()


def test_sgd_kernel_bitexact():
    lib = _lib.load()
    n = 1_000_003
    rng = np.random.default_rng(1)
    th = rng.standard_normal(n).astype(np.float32)
    v = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    lr, mu = np.float32(0.1), np.float32(0.9)
    T = [torch.from_numpy(a.copy()).cuda() for a in (th, v, g)]
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.ds_sgd_momentum(T[0].data_ptr(), T[1].data_ptr(), T[2].data_ptr(), float(lr), float(mu), n, None,
                                   flag.data_ptr(), _lib.stream_ptr()))
    torch.cuda.synchronize()
    v_ref = (v * mu).astype(np.float32) + g
    th_ref = th - (lr * v_ref).astype(np.float32)
    assert np.array_equal(T[1].cpu().numpy(), v_ref)
    assert np.array_equal(T[0].cpu().numpy(), th_ref)
    assert flag.item() == 0
    T[2][5] = float("nan")
    _lib.check(lib.ds_sgd_momentum(T[0].data_ptr(), T[1].data_ptr(), T[2].data_ptr(), float(lr), float(mu), n, None,
                                   flag.data_ptr(), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert flag.item() == 1


def test_mix_kernel_pair_sum_exact():
    lib = _lib.load()
    n = 777_777
    rng = np.random.default_rng(2)
    a = rng.standard_normal(n).astype(np.float32)
    b = (rng.standard_normal(n) * 1e3).astype(np.float32)
    A, Bt = torch.from_numpy(a.copy()).cuda(), torch.from_numpy(b.copy()).cuda()
    _lib.check(lib.ds_adpsgd_mix(A.data_ptr(), Bt.data_ptr(), n, _lib.stream_ptr()))
    torch.cuda.synchronize()
    m = ((a + b) / np.float32(2)).astype(np.float32)
    assert np.array_equal(A.cpu().numpy(), m) and np.array_equal(Bt.cpu().numpy(), m)
    # identical value on both sides => pair sum preserved bit-exactly (test_adpsgd.py:34-41)
    assert np.array_equal(A.cpu().numpy() + Bt.cpu().numpy(), (a + b).astype(np.float32))


@pytest.mark.parametrize("world,chunks,n", [(2, None, 100_003), (3, 7, 100_003), (4, None, 100_003),
                                            (8, 16, 100_003), (2, 4, 10), (3, 5, 13)])
def test_group_reduce_canonical_order(world, chunks, n):
    """n=10 / 4 chunks: the last chunk [9, 10) holds no aligned float4 (its
    edge ranges used to overlap and apply the step twice)."""
    lib = _lib.load()
    chunks = chunks or world
    rng = np.random.default_rng(world)
    gs = [rng.standard_normal(n).astype(np.float32) * (10.0 ** k) for k in range(world)]
    th = rng.standard_normal(n).astype(np.float32)
    v = rng.standard_normal(n).astype(np.float32)
    G = [torch.from_numpy(x).cuda() for x in gs]
    TH = [torch.from_numpy(th.copy()).cuda() for _ in range(world)]
    V = [torch.from_numpy(v.copy()).cuda() for _ in range(world)]
    ptrs = ctypes_arr
    for r in range(world):
        _lib.check(lib.ds_group_reduce(world, r, ptrs(G), ptrs(TH), ptrs(V), None, n, chunks, 0.1, 0.9, 0, 0.0,
                                       _lib.stream_ptr()))
    torch.cuda.synchronize()
    size = -(-n // chunks)
    mean = np.empty(n, np.float32)
    for j in range(chunks):
        lo, hi = min(j * size, n), min((j + 1) * size, n)
        o = j % world
        s = gs[o][lo:hi].copy()
        for k in range(1, world):
            s = (s + gs[(o + k) % world][lo:hi]).astype(np.float32)
        mean[lo:hi] = s / np.float32(world)
    v_ref = (v * np.float32(0.9)).astype(np.float32) + mean
    th_ref = th - (np.float32(0.1) * v_ref).astype(np.float32)
    for r in range(world):
        assert np.array_equal(TH[r].cpu().numpy(), th_ref)
        assert np.array_equal(V[r].cpu().numpy(), v_ref)


def ctypes_arr(ts):
    import ctypes

    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


@pytest.mark.parametrize("layers,B,T,classes", [(3, 32, 5, 512), (2, 256, 21, 1024)])
def test_fused_train_step_equals_gradient_then_sgd(layers, B, T, classes):
    """ds_blstm_train_step (per-layer SGD beside the next BPTT) is bit-identical
    to ds_blstm_fwd_bwd followed by ds_sgd_momentum, over several steps (so the
    refreshed snapshot, padded W_ih0 and bias copies are exercised too)."""
    obj = BlstmObjective(layers=layers, classes=classes, frames=T)
    spec = _spec(obj)
    x, y, _, _ = O.make_dataset(spec, 3 * B, seed=7)
    w = O.initial_weights(spec, 7)
    data = DeviceDataset(x, y)
    A = Learner(obj, data, max_batch=B, theta0=w)
    R = Learner(obj, data, max_batch=B, theta0=w)
    rng = np.random.default_rng(1)
    for step, lr in enumerate((0.05, 0.02, 0.08)):
        batch = rng.permutation(len(x))[:B]
        A.train_step(batch, lr)
        R.gradient(batch)
        R.sgd_step(lr)
        A.check_finite()
        R.check_finite()
        assert A.mean_loss() == R.mean_loss(), step
        for name in ("grad", "vel", "theta"):
            a, r = getattr(A, name), getattr(R, name)
            assert torch.equal(a, r), (step, name, (a - r).abs().max().item())
    A.close()
    R.close()


def test_unfused_output_layer_matches_fused(tmp_path):
    """DS_NO_FUSED_CE=1 selects the GEMM-epilogue output layer (soft-max
    statistics / gradient epilogues + separate dW_o, dZ GEMMs) instead of the
    CTA-pair statistics and soft-max/dZ kernels: both paths agree within the
    BF16 tolerance (the switch is read once per process: subprocess)."""
    import os
    import subprocess
    import sys

    script = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from oracle import blstm_ref as O
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner
obj = BlstmObjective(layers=1, classes=1280, frames=5)
spec = O.BlstmSpec(layers=1, input_dim=obj.input_dim, hidden=512, bottleneck=obj.bottleneck, classes=1280, frames=5)
x, y, _, _ = O.make_dataset(spec, 80, seed=3)
w = O.initial_weights(spec, 3)
L = Learner(obj, DeviceDataset(x, y), max_batch=64, theta0=w)
L.gradient(np.arange(64))
np.save(sys.argv[1], np.concatenate([[L.mean_loss()], L.grad.double().cpu().numpy()]))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_val in ("0", "1"):
        out = tmp_path / f"g{env_val}.npy"
        env = dict(os.environ, DS_NO_FUSED_CE=env_val)
        subprocess.run([sys.executable, "-c", script, str(out)], check=True, env=env, timeout=300)
        outs.append(np.load(out))
    a, b = outs
    assert abs(a[0] - b[0]) <= 1e-3 * abs(a[0]), (a[0], b[0])
    ga, gb = a[1:], b[1:]
    rel = np.linalg.norm(ga - gb) / np.linalg.norm(gb)
    assert rel <= 1e-2, rel


@pytest.mark.parametrize("layers,B,T,classes,bott,din", [
    (1, 1, 4, 512, 256, 260),     # one sequence: batch tiles of one row
    (2, 5, 1, 256, 256, 260),     # one frame: the recurrences have a single step (no recurrent term)
    (1, 17, 3, 384, 64, 40),      # bottleneck 64 (GEMM-epilogue soft-max path), narrow input
    (1, 300, 2, 128, 128, 260),   # batch > one recurrent launch's 256 rows: two sub-launches
])
def test_fwd_bwd_edge_shapes_match_oracle(layers, B, T, classes, bott, din):
    """Edge shapes of the same path against the float64 oracle (tolerances as above)."""
    obj = BlstmObjective(layers=layers, classes=classes, frames=T, bottleneck=bott, input_dim=din)
    spec = O.BlstmSpec(layers=layers, input_dim=din, hidden=512, bottleneck=bott, classes=classes, frames=T)
    assert spec.param_dim == obj.param_dim
    x, y, _, _ = O.make_dataset(spec, B + 2, seed=11)
    w = O.initial_weights(spec, 11)
    batch = np.arange(B)
    xb = torch.from_numpy(x).bfloat16().double().numpy()
    loss_ref, g_ref = O.loss_and_grad(spec, w, xb[batch], y[batch])
    L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=w)
    L.gradient(batch)
    L.check_finite()
    loss = L.mean_loss()
    g = L.grad.double().cpu().numpy()
    assert abs(loss - loss_ref) <= 5e-3 * abs(loss_ref), (loss, loss_ref)
    for k, v in offsets(obj).items():
        if k == "total":
            continue
        o, shape = v
        n = int(np.prod(shape))
        a, r = g[o:o + n], g_ref[o:o + n]
        if np.linalg.norm(r) == 0:
            continue
        rel = np.linalg.norm(a - r) / np.linalg.norm(r)
        cos = float(a @ r / max(np.linalg.norm(a) * np.linalg.norm(r), 1e-30))
        assert rel <= 2.5e-2 and cos >= 0.9995, (k, rel, cos)
    L.close()


def test_loss_async_matches_mean_loss():
    """Learner.loss_async (pinned ring, read after the next step is issued) gives
    each step's own mean loss."""
    obj = BlstmObjective(layers=1, classes=256, frames=3)
    spec = _spec(obj)
    x, y, _, _ = O.make_dataset(spec, 64, seed=2)
    L = Learner(obj, DeviceDataset(x, y), max_batch=32, theta0=O.initial_weights(spec, 2))
    futs, refs = [], []
    for k in range(6):
        L.train_step(np.arange(k, k + 32) % 64, 0.05)
        futs.append(L.loss_async())
        if k >= 1:
            refs.append(futs[k - 1]())
    refs.append(futs[-1]())
    R = Learner(obj, DeviceDataset(x, y), max_batch=32, theta0=O.initial_weights(spec, 2))
    for k in range(6):
        R.train_step(np.arange(k, k + 32) % 64, 0.05)
        assert R.mean_loss() == refs[k], k
    L.close()
    R.close()
