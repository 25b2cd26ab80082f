"""One-process-per-GPU P2P path (paper_1904_04956_b200/p2p.py, csrc/p2p.cu).

CPU: the partner schedule is the reference Topology and a perfect matching
every iteration (so lock-step ADPSGD pairs never overlap).
GPU: two processes share cuda:0 through CUDA IPC (the same mechanism that maps
a neighbour GPU's memory over NVLink); the sharded SSGD step and the pairwise
mix must equal float32 restatements of the reference arithmetic bit for bit,
and every replica must hold identical weights afterwards."""

import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1904_04956_b200.p2p import adpsgd_partner, hadpsgd_layout


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partner_schedule_is_topology_matching(world):
    from paper_1904_04956_b200.schedule import Topology

    topo = Topology(world)
    for it in range(1, 9):
        p = [adpsgd_partner(r, world, it) for r in range(world)]
        assert sorted(p) == list(range(world))            # a permutation ...
        assert all(p[p[r]] == r and p[r] != r for r in range(world))  # ... of disjoint pairs
        for s in topo.senders():
            assert p[s - 1] == topo.partner(s, it) - 1


def test_partner_schedule_matches_reference(ref):
    from distsgd.engines.common import Topology as RefTopology

    for world in (2, 4, 8):
        t = RefTopology(world)
        for it in range(1, 7):
            for s in range(1, world + 1, 2):
                assert adpsgd_partner(s - 1, world, it) == t.partner(s, it) - 1


def test_hadpsgd_layout():
    assert [hadpsgd_layout(r, 2, 4) for r in range(8)] == [(0, 0), (0, 1), (0, 2), (0, 3), (1, 0), (1, 1), (1, 2),
                                                         (1, 3)]
    with pytest.raises(ValueError):
        hadpsgd_layout(8, 2, 4)


# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import blstm_ref as O
    from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner
    from paper_1904_04956_b200.p2p import PeerGroup

    torch.cuda.set_device(0)
    obj = BlstmObjective(layers=1, bottleneck=64, classes=64, frames=3)
    spec = O.BlstmSpec(layers=1, input_dim=260, hidden=512, bottleneck=64, classes=64, frames=3)
    x, y, _, _ = O.make_dataset(spec, 32, seed=0)
    w0 = O.initial_weights(spec, 0)
    L = Learner(obj, DeviceDataset(x, y), max_batch=8, theta0=w0)
    G = PeerGroup(L, rank, world, timeout_s=120.0)
    out = {}
    # --- SSGD: same weights, different batches -> identical replicas
    L.gradient(np.arange(8) + 8 * rank)
    L.stream.synchronize()
    out["g"] = L.grad.cpu().numpy()
    out["theta0"] = L.theta.cpu().numpy()
    G.ssgd_step(0.05)
    G.check()
    out["theta_ssgd"] = L.theta.cpu().numpy()
    from paper_1904_04956_b200 import _lib

    snap = torch.empty(obj.param_dim, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    _lib.check(lib.ds_device_copy(snap.data_ptr(), lib.ds_blstm_snapshot_ptr(L.handle), obj.param_dim * 2,
                                  L.stream.cuda_stream))
    L.stream.synchronize()
    out["snap_ssgd"] = snap.float().cpu().numpy()
    # the step refreshed the bf16 operand snapshot: the loss on it equals the
    # loss after an explicit re-cast of theta (and is the same on both ranks)
    L.loss(np.arange(8))
    L.stream.synchronize()
    out["loss_step_snap"] = np.float32(L.loss_sum.item())
    L.snapshot()
    L.loss(np.arange(8))
    L.stream.synchronize()
    out["loss_recast"] = np.float32(L.loss_sum.item())
    # --- ADPSGD mix: different weights -> both hold (a + b) / 2
    with torch.cuda.stream(L.stream):
        L.theta.mul_(1.0 + 0.25 * (rank + 1)).add_(0.001 * (rank + 1))
    L.stream.synchronize()
    out["theta_pre_mix"] = L.theta.cpu().numpy()
    G.mix(1 - rank)
    G.check()
    out["theta_mix"] = L.theta.cpu().numpy()
    G.close()
    L.close()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_ipc_ssgd_and_mix_bit_exact():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        r = [dict(np.load(os.path.join(d, f"r{i}.npz"))) for i in range(2)]
    # SSGD: canonical-order chunk sums (owner first), / world, v = 0*mu + g, theta - lr*v (float32)
    P = r[0]["g"].shape[0]
    chunk = -(-P // 2)
    g0, g1 = r[0]["g"], r[1]["g"]
    s = np.empty(P, np.float32)
    s[:chunk] = g0[:chunk] + g1[:chunk]      # chunk 0: owner 0 then 1
    s[chunk:] = g1[chunk:] + g0[chunk:]      # chunk 1: owner 1 then 0
    gm = s / np.float32(2)
    v = np.float32(0.9) * np.zeros(P, np.float32) + gm
    want = r[0]["theta0"] - np.float32(0.05) * v
    assert np.array_equal(r[0]["theta_ssgd"], r[1]["theta_ssgd"])
    assert np.array_equal(r[0]["theta_ssgd"], want)
    bf = torch.from_numpy(want).bfloat16().float().numpy()
    for k in (0, 1):
        bad = np.nonzero(r[k]["snap_ssgd"] != bf)[0]
        assert bad.size == 0, (k, bad.size, bad[:3], bad[-3:], P)
    for k in (0, 1):
        assert r[k]["loss_step_snap"] == r[k]["loss_recast"]
    assert r[0]["loss_step_snap"] == r[1]["loss_step_snap"]
    # mix
    m = (r[0]["theta_pre_mix"] + r[1]["theta_pre_mix"]) * np.float32(0.5)
    assert np.array_equal(r[0]["theta_mix"], m) and np.array_equal(r[1]["theta_mix"], m)


def _bench(nproc, *extra, timeout=600):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", str(nproc), "--no-cpu", "--same-device",
           *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("strategy,nproc,mode", [("ssgd", 2, "overlap"), ("ssgd", 2, "after"), ("adpsgd", 2, "async"),
                                                 ("adpsgd", 2, "fused"), ("adpsgd", 2, "lockstep"),
                                                 ("hadpsgd", 4, "async")])
def test_bench_self_spawn_same_device(strategy, nproc, mode):
    """`bench.py --gpus N` spawns its own ranks (no external torchrun) and runs
    every strategy / mode end to end with all ranks on cuda:0 (functional:
    the ranks time-slice one GPU)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    mflag = ["--ssgd-mode", mode] if strategy == "ssgd" else ["--adpsgd-mode", mode]
    rec = _bench(nproc, "--steps", "3", "--warmup", "3", "--n-seq", "512", "--batch", "32", "--layers", "2",
                 "--classes", "1024", "--strategy", strategy, "--groups", "2", *mflag)
    assert rec["n_gpus"] == nproc and rec["config"]["strategy"] == strategy and rec["config"]["mode"] == mode
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0 and len(rec["per_rank_ms"]) == nproc


@pytest.mark.gpu
def test_async_adpsgd_is_straggler_immune():
    """One learner 2x slower per step (injected on the real clock, as the
    reference's DelayModel slowdowns / harness straggler sweep,
    runtime.py:47-91, harness.py:141-158): with the asynchronous protocol the
    other learners' step time stays within 15 % of the no-straggler run
    ("immune to the straggler problem"); the lock-step pairing
    drags the straggler's partners down."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    common = ["--steps", "15", "--warmup", "3", "--n-seq", "512", "--batch", "16", "--layers", "1", "--classes",
              "256", "--strategy", "adpsgd", "--base-sleep", "0.03"]
    base = _bench(4, *common)
    slow = _bench(4, *common, "--straggler-rank", "1", "--straggler-sleep", "0.03")
    lock = _bench(4, *common, "--adpsgd-mode", "lockstep", "--straggler-rank", "1", "--straggler-sleep", "0.03")
    print("per-rank ms: base", base["per_rank_ms"], "straggler", slow["per_rank_ms"], "lockstep", lock["per_rank_ms"])
    others = [0, 2, 3]
    for r in others:
        assert slow["per_rank_ms"][r] <= 1.15 * base["per_rank_ms"][r], (r, slow["per_rank_ms"], base["per_rank_ms"])
    assert slow["per_rank_ms"][1] >= 1.6 * base["per_rank_ms"][1]  # the straggler really was slower
    assert max(lock["per_rank_ms"][r] for r in others) >= 1.5 * max(base["per_rank_ms"][r] for r in others)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy,nproc", [("ssgd", 2), ("adpsgd", 2), ("hadpsgd", 4)])
def test_bench_multiprocess_p2p_same_device(strategy, nproc):
    """bench.py's one-process-per-GPU path (torchrun, P2P transport) runs end
    to end with both ranks on cuda:0 and prints one JSON line (functional
    check: ranks time-slice one GPU, the value is not a scaling number)."""
    import json
    import subprocess
    import sys

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus",
           str(nproc), "--steps", "3", "--warmup", "3", "--no-cpu", "--n-seq", "1024", "--batch", "64",
           "--same-device", "--strategy", strategy, "--groups", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == nproc and rec["config"]["strategy"] == strategy and rec["config"]["transport"] == "p2p"
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0


def _worker_async(rank, world, port, outdir):
    """Fused per-layer SSGD group step vs gradient + ssgd_step; asynchronous
    ADPSGD exchange (sender-initiated, receiver lock); fused update+mix."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import blstm_ref as O
    from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner
    from paper_1904_04956_b200.p2p import PeerGroup

    torch.cuda.set_device(0)
    obj = BlstmObjective(layers=2, bottleneck=64, classes=128, frames=3)
    spec = O.BlstmSpec(layers=2, input_dim=260, hidden=512, bottleneck=64, classes=128, frames=3)
    x, y, _, _ = O.make_dataset(spec, 40, seed=1)
    w0 = O.initial_weights(spec, 1)
    L = Learner(obj, DeviceDataset(x, y), max_batch=8, theta0=w0)
    G = PeerGroup(L, rank, world, timeout_s=120.0)
    out = {}
    batches = [np.arange(8) + 8 * rank, np.arange(8) + 16 + 8 * rank]
    # (1) two SSGD steps, per-layer overlapped inside the fused step, chunk_count 5
    G.attach_fused_ssgd(chunk_count=5)
    for k, b in enumerate(batches):
        L.train_step(b, 0.05 * (k + 1))
    G.check()
    L.check_finite()
    out["theta_fused"] = L.theta.cpu().numpy()
    out["vel_fused"] = L.vel.cpu().numpy()
    G.detach_fused_ssgd()
    dist.barrier()
    # (2) the same two steps as gradient + whole-vector sharded step
    L.set_weights(w0)
    with torch.cuda.stream(L.stream):
        L.vel.zero_()
    for k, b in enumerate(batches):
        L.gradient(b)
        G.ssgd_step(0.05 * (k + 1), chunk_count=5)
    G.check()
    out["theta_unfused"] = L.theta.cpu().numpy()
    out["vel_unfused"] = L.vel.cpu().numpy()
    dist.barrier()
    # (3) asynchronous exchange: rank 0 (learner 1, sender) mixes into rank 1 (receiver)
    with torch.cuda.stream(L.stream):
        L.theta.mul_(1.0 + 0.5 * rank).add_(0.01 * rank)
    L.stream.synchronize()
    out["pre"] = L.theta.cpu().numpy()
    dist.barrier()
    if rank == 0:
        G.exchange_async(1)
        G.ack_gate()
    G.check()
    dist.barrier()
    out["post_mix"] = L.theta.cpu().numpy()
    dist.barrier()
    # (4) receiver update racing the sender's exchange: atomic either way
    L.gradient(batches[0])
    L.stream.synchronize()
    out["pre2"] = L.theta.cpu().numpy()
    out["vel_pre2"] = L.vel.cpu().numpy()
    out["g2"] = L.grad.cpu().numpy()
    dist.barrier()
    if rank == 0:
        G.exchange_async(1)
        G.ack_gate()
    else:
        G.locked_update(0.03)
    G.check()
    dist.barrier()
    out["post_race"] = L.theta.cpu().numpy()
    dist.barrier()
    # (5) fused sender update + mix (ds_update_mix)
    L.gradient(batches[1])
    L.stream.synchronize()
    out["pre3"] = L.theta.cpu().numpy()
    out["vel_pre3"] = L.vel.cpu().numpy()
    out["g3"] = L.grad.cpu().numpy()
    dist.barrier()
    if rank == 0:
        G.update_exchange_async(1, 0.02)
    G.check()
    dist.barrier()
    out["post_fused"] = L.theta.cpu().numpy()
    from paper_1904_04956_b200 import _lib

    snap = torch.empty(obj.param_dim, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    _lib.check(lib.ds_device_copy(snap.data_ptr(), lib.ds_blstm_snapshot_ptr(L.handle), obj.param_dim * 2,
                                  L.stream.cuda_stream))
    L.stream.synchronize()
    out["snap_fused"] = snap.float().cpu().numpy()
    G.close()
    L.close()
    np.savez(os.path.join(outdir, f"a{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_fused_ssgd_and_async_adpsgd():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker_async, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        r = [dict(np.load(os.path.join(d, f"a{i}.npz"))) for i in range(2)]
    f32 = np.float32
    # (1) == (2): the per-layer overlapped SSGD step is bit-identical to the whole-vector one
    for k in (0, 1):
        assert np.array_equal(r[k]["theta_fused"], r[k]["theta_unfused"])
        assert np.array_equal(r[k]["vel_fused"], r[k]["vel_unfused"])
    assert np.array_equal(r[0]["theta_fused"], r[1]["theta_fused"])
    # (3) one-sided exchange: the identical mean in both learners
    m = (r[0]["pre"] + r[1]["pre"]) * f32(0.5)
    assert np.array_equal(r[0]["post_mix"], m) and np.array_equal(r[1]["post_mix"], m)
    # (4) the receiver's update and the sender's mix never interleave: either the
    # mix saw the updated receiver or the update came after the mix — for ALL elements
    a, b = r[0]["pre2"], r[1]["pre2"]
    v = (r[1]["vel_pre2"] * f32(0.9)).astype(f32) + r[1]["g2"]
    b_upd = b - (f32(0.03) * v).astype(f32)
    mix_after = (a + b_upd) * f32(0.5)
    mix_before = (a + b) * f32(0.5)
    s_after = np.array_equal(r[0]["post_race"], mix_after) and np.array_equal(r[1]["post_race"], mix_after)
    s_before = np.array_equal(r[0]["post_race"], mix_before) and np.array_equal(
        r[1]["post_race"], mix_before - (f32(0.03) * v).astype(f32))
    assert s_after or s_before
    # (5) fused: t' = theta - lr (mu v + g); snapshot bf16(t'); mean into both
    a, b = r[0]["pre3"], r[1]["pre3"]
    v = (r[0]["vel_pre3"] * f32(0.9)).astype(f32) + r[0]["g3"]
    t = a - (f32(0.02) * v).astype(f32)
    m = (t + b) * f32(0.5)
    assert np.array_equal(r[0]["post_fused"], m) and np.array_equal(r[1]["post_fused"], m)
    assert np.array_equal(r[0]["snap_fused"], torch.from_numpy(t).bfloat16().float().numpy())
