#!/usr/bin/env python
"""bench.py — training frames/s of the paper BLSTM on B200 (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

N = 1 : config "paper BLSTM ... SSGD batch 256 on 1 B200" — the reference's
        single-learner path run_single (engines/single.py:49-55): gather ->
        fwd/bwd -> learning_rate -> sgd_step, per minibatch of 256 21-frame
        sequences drawn from epoch_minibatches.
N > 1 : one rank per GPU (torchrun), per-learner batch B (weak scaling),
        --strategy ssgd (default) | adpsgd | hadpsgd:
          ssgd     every rank's gradient is reduced in the reference's
                   canonical chunk order, /world, momentum SGD on the owned
                   chunk and theta all-gathered (ds_shard_step);
          adpsgd   local momentum SGD, then ADPSGD pairwise averaging with
                   the ring Topology partner of this iteration (ds_pair_mix),
                   lock-step: every learner updates once per step;
          hadpsgd  --groups groups: SSGD inside a group, then member r of a
                   group averages with member r of the partner group.
        --transport p2p (default): libds kernels over CUDA-IPC-mapped peer
        memory (NVLink P2P) with device barriers; --transport nccl: the same
        schedule with torch.distributed/NCCL collectives (comparison only).
`value` is device-timed (CUDA events on the learner stream, inputs resident
in HBM, max over ranks); `e2e` goes through the public Learner API with the
minibatch indices copied host->device and the loss read back every step.
`--impl reference` times the CPU oracle port (oracle/blstm_ref.py, float64
numpy, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training frames/sec at 1/2/4/8 B200 per strategy (SSGD/ADPSGD/H-ADPSGD)"
UNIT = "frames/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), float(
            d["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    (sub-millisecond queries, so even a ~50 ms region gets many samples),
    falling back to `nvidia-smi` polling when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv) -> None:
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                              nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            self._stop.wait(0.002)

    def _run_smi(self) -> None:
        fields = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                p = [x.strip() for x in out.stdout.strip().split(",")]
                self.rows.append((float(p[0]), float(p[1]), int(p[2], 16)))
            except Exception:
                pass
            self._stop.wait(0.05)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
        except Exception:
            self._run_smi()
            return
        try:
            self._run_nvml(nv)
        finally:
            nv.nvmlShutdown()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.01)  # the sampler is running before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for _, _, m in self.rows for name, bit in self.REASONS if m & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows)}


def make_data(obj, n_seq: int, seed: int = 0):
    """Synthetic SWB-shaped data: x ~ N(0,1), y ~ U{0..C-1}."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n_seq, obj.frames, obj.input_dim), dtype=np.float32)
    y = rng.integers(0, obj.classes, size=(n_seq, obj.frames), dtype=np.int64)
    n_held = n_seq // 10
    return x, y, np.arange(n_seq - n_held)


# ---------------------------------------------------------------------------
def cpu_reference(obj, batch: int, steps: int, warmup: int, seed: int = 0):
    """The CPU oracle port timed on the host cores (float64 numpy, BLAS uses
    every host thread).  Returns (frames/s, seconds per step)."""
    from oracle import blstm_ref as O

    spec = O.BlstmSpec(layers=obj.layers, input_dim=obj.input_dim, hidden=512, bottleneck=obj.bottleneck,
                       classes=obj.classes, frames=obj.frames)
    rng = np.random.default_rng(seed)
    w = O.initial_weights(spec, seed)
    v = np.zeros_like(w)
    times = []
    for i in range(warmup + steps):
        x = rng.standard_normal((batch, spec.frames, spec.input_dim))
        y = rng.integers(0, spec.classes, size=(batch, spec.frames))
        t0 = time.perf_counter()
        _, g = O.loss_and_grad(spec, w, x, y)
        v *= 0.9
        v += g
        w = w - 0.1 * v
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    sec = sum(times) / len(times)
    return batch * spec.frames / sec, sec


def library_baseline(obj, B: int, steps: int = 10, warmup: int = 3):
    """Same-box library path at the same config (SURVEY §2.1 "the bar"):
    cuDNN bidirectional nn.LSTM + nn.Linear bottleneck/output +
    F.cross_entropy + torch.optim.SGD(momentum, fused) under bf16 autocast,
    inputs resident, CUDA-event timed.  Returns a dict for the bench line."""
    import torch
    import torch.nn as nn
    import torch.nn.functional as F

    dev = torch.device("cuda", torch.cuda.current_device())
    T, D, C = obj.frames, obj.input_dim, obj.classes
    torch.manual_seed(0)
    lstm = nn.LSTM(D, 512, num_layers=obj.layers, bidirectional=True).to(dev)
    bott = nn.Linear(1024, obj.bottleneck).to(dev)
    outl = nn.Linear(obj.bottleneck, C).to(dev)
    params = list(lstm.parameters()) + list(bott.parameters()) + list(outl.parameters())
    try:
        opt = torch.optim.SGD(params, lr=0.1, momentum=0.9, fused=True)
    except Exception:  # pragma: no cover
        opt = torch.optim.SGD(params, lr=0.1, momentum=0.9, foreach=True)
    x = torch.randn(T, B, D, device=dev)
    y = torch.randint(0, C, (T * B,), device=dev)
    res = {}
    for dt_name, dt in (("bf16", torch.bfloat16), ("fp16", torch.float16)):
        try:
            def step():
                opt.zero_grad(set_to_none=True)
                with torch.autocast("cuda", dtype=dt):
                    h, _ = lstm(x)
                    logits = outl(bott(h))
                loss = F.cross_entropy(logits.float().view(-1, C), y)
                loss.backward()
                opt.step()
                return loss

            for _ in range(warmup):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            res = {"value": round(B * T / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 4),
                   "dtype": dt_name, "steps": steps,
                   "what": "torch.nn.LSTM (cuDNN, 6x bidirectional 512) + Linear 1024->256 + Linear 256->32000 + "
                           "F.cross_entropy + torch.optim.SGD(momentum=0.9, fused) under autocast, B=%d" % B}
            break
        except Exception as exc:  # pragma: no cover - recorded, not fatal
            res = {"unavailable": f"{dt_name}: {type(exc).__name__}: {exc}"[:300]}
    del lstm, bott, outl, opt, params
    torch.cuda.empty_cache()
    return res


def engine_epoch(obj, B: int, x_host) -> dict:
    """The drop-in strategy API end to end: engines.run_single (the
    reference's run_single signature, engines/single.py:14-74) over one epoch
    of the bench dataset on the real clock — host index lists, the fused
    step, the epoch's held-out evaluation and the weight read-back included.
    Reports the engine's own MetricsRecord.frames_per_s."""
    from paper_1904_04956_b200 import engines as E
    from paper_1904_04956_b200.backend import GpuBackend
    from paper_1904_04956_b200.objective import Dataset
    from paper_1904_04956_b200.runtime import RealClock
    from paper_1904_04956_b200.schedule import baseline_schedule

    x, y, train = x_host
    held = np.arange(len(train), len(x))
    data = Dataset(x, y, train, held)
    be = GpuBackend(obj, data, max_batch=B)
    t0 = time.perf_counter()
    res = E.run_single(obj, data, baseline_schedule(0.1), epochs=2, batch_size=B, seed=0, clock=RealClock(),
                       backend=be)
    wall = time.perf_counter() - t0
    be.close()
    r = res.records[-1]  # epoch 2: the step graphs (full and short final batch) are captured
    return {"value": round(r.frames_per_s, 1), "unit": UNIT, "epoch_wall_s": round(r.epoch_wall_s, 4),
            "minibatches": r.minibatch_counts[0], "heldout_sequences": int(len(held)),
            "call_wall_s": round(wall, 3),
            "what": "engines.run_single, epoch 2 of the bench dataset on the real clock (per-epoch held-out "
                    "loss and finiteness check included in the call, not in the epoch wall)"}


def run_reference_arm(args, rank: int, world: int = 1):
    from paper_1904_04956_b200.blstm import BlstmObjective

    if rank != 0:
        return
    obj = BlstmObjective()
    cb = args.batch  # the same config as our arm (config 2: B = 256)
    steps = max(1, min(args.steps, args.ref_max_steps))
    warm = max(0, min(args.warmup, 1))
    fps, sec = cpu_reference(obj, cb, steps, warm)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(fps, 2), "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": round(sec * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(obj, cb, world, "single" if world == 1 else args.strategy, args,
                               args.groups, max(1, world // max(1, args.groups))),
        "reference_note": ("the float64 CPU port of one learner's training step on all host cores; with N "
                           "learners the host's aggregate is the same (the learners would share the cores)"),
        "cpu_baseline": {"value": round(fps, 2), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{steps} step(s) of B={cb} sequences x 21 frames, paper-size model, float64"},
        "e2e": {"value": round(fps, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_config(obj, B: int, world: int, strategy: str, args, ngroups: int = 1, gsize: int = 1) -> dict:
    """The workload description shared by both arms (same keys and values,
    so the driver can match the reference arm's line to ours)."""
    return {"workload": ("paper BLSTM run_single step, batch 256 (config 2)" if world == 1 else
                         f"paper BLSTM {strategy.upper()}, {B}/learner, transport={args.transport}"
                         + (f", {ngroups} groups x {gsize}" if strategy == "hadpsgd" else "")),
            "layers": obj.layers, "cells": 1024, "bottleneck": obj.bottleneck, "classes": obj.classes,
            "input_dim": obj.input_dim, "frames": obj.frames, "batch_per_learner": B, "global_batch": B * world,
            "strategy": strategy, "transport": args.transport if world > 1 else None,
            "mode": (args.ssgd_mode if strategy == "ssgd" else args.adpsgd_mode
                     if strategy in ("adpsgd", "hadpsgd") else None),
            "straggler": ({"rank": args.straggler_rank, "extra_sleep_s": args.straggler_sleep}
                          if args.straggler_sleep > 0 else None),
            "l2_policy": "per-step working set ~1.2 GB (activations, 344 MB dlogits) >> 126 MB L2; no flush",
            "parallelism": f"dp{world}"}


# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch

    from paper_1904_04956_b200.blstm import (BlstmObjective, DeviceDataset, Learner, initial_weights,
                                             training_flops_per_frame)
    from paper_1904_04956_b200.schedule import baseline_schedule, epoch_minibatches, learning_rate

    if args.same_device:  # functional check of the multi-process path on a one-GPU box (time-sliced)
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist

        if args.same_device:
            dist.init_process_group("gloo")
            red_dev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    obj = BlstmObjective(layers=args.layers, classes=args.classes)
    B = args.batch
    T = obj.frames
    x, y, train = make_data(obj, args.n_seq, seed=0)
    data = DeviceDataset(x, y, device=local_rank)
    del x
    L = Learner(obj, data, max_batch=B, device=local_rank, theta0=initial_weights(obj, 0))
    sched = baseline_schedule(0.1)
    # the run_single draw order; rank r of an SSGD group takes every world-th batch (static_partition)
    from paper_1904_04956_b200.distributed import rank_batches

    mine = [b for b in rank_batches(train, B, 0, 1, rank, world) if len(b) == B]
    q = len(mine)
    idx_dev = torch.from_numpy(np.stack(mine)).to(torch.device("cuda", local_rank))
    stream = L.stream
    P = obj.param_dim
    strategy = "single" if world == 1 else args.strategy
    if strategy in ("adpsgd", "hadpsgd") and world % 2:
        raise SystemExit("adpsgd / hadpsgd need an even number of learners")
    group = None
    if world > 1 and args.transport == "p2p":
        from paper_1904_04956_b200.p2p import PeerGroup

        group = PeerGroup(L, rank, world)
        if strategy == "ssgd" and args.ssgd_mode == "overlap":
            group.attach_fused_ssgd()
    from paper_1904_04956_b200.p2p import adpsgd_partner

    ngroups = args.groups if strategy == "hadpsgd" else 1
    gsize = world // max(1, ngroups)
    if strategy == "hadpsgd" and (ngroups < 2 or world % ngroups or ngroups % 2):
        raise SystemExit("hadpsgd needs an even group count dividing the learner count")
    peer_buf = torch.empty_like(L.theta) if (world > 1 and args.transport == "nccl" and strategy != "ssgd") else None

    def nccl_mix(peer: int):
        ops = [dist.P2POp(dist.isend, L.theta, peer), dist.P2POp(dist.irecv, peer_buf, peer)]
        with torch.cuda.stream(stream):
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            L.theta.add_(peer_buf).mul_(0.5)
        L.snapshot()

    from paper_1904_04956_b200.distributed import step_plan

    plan1 = step_plan(strategy, rank, world, 1, ngroups)
    members, is_sender = list(plan1.members), plan1.initiates
    straggle = args.straggler_sleep if rank == args.straggler_rank else 0.0

    def step(k: int, host: bool = False):
        """One learner iteration of the strategy (k = this rank's update count - 1);
        host=True: the minibatch indices come from host memory (public API, e2e)."""
        j = k % q
        lr = learning_rate(sched, 1, j, q)

        def grad():
            L.gradient(mine[j]) if host else L.gradient_device(idx_dev[j], B)

        def fused(lr):
            L.train_step(mine[j], lr) if host else L.train_step(idx_dev[j], lr, device_idx=True)

        if args.base_sleep > 0 or straggle > 0:  # injected compute time / slowdown on the real clock
            time.sleep(args.base_sleep + straggle)  # (DelayModel base_compute_s / slowdowns, runtime.py:47-91)
        if strategy == "single":  # gradient + momentum SGD fused in one graph
            fused(lr)
            return
        if strategy == "adpsgd" and args.adpsgd_mode == "lockstep" or group is None:
            if strategy == "ssgd":
                grad()
                with torch.cuda.stream(stream):
                    dist.all_reduce(L.grad)
                    L.grad.div_(world)
                L.sgd_step(lr)
                return
            if strategy == "hadpsgd":
                raise SystemExit("hadpsgd is implemented on the p2p transport only")
            fused(lr)  # lock-step comparison: pair barriers every step
            peer = adpsgd_partner(rank, world, k + 1)
            group.mix(peer) if group is not None else nccl_mix(peer)
            return
        if strategy == "ssgd":
            if args.ssgd_mode == "overlap":  # per-layer group sync inside the fused step (ds_blstm_set_group)
                fused(lr)
            else:
                grad()
                group.ssgd_step(lr)
            return
        grad()
        # asynchronous ADPSGD / H-ADPSGD (engines/adpsgd.py:115-288): senders initiate
        plan = step_plan(strategy, rank, world, k + 1, ngroups)
        if plan.initiates:
            group.ack_gate()  # the previous exchange was acknowledged
            if strategy == "hadpsgd":
                group.ssgd_step(lr, members=list(plan.members))
            elif args.adpsgd_mode == "fused":
                group.update_exchange_async(plan.partner, lr)
                return
            else:
                L.sgd_step(lr)
            group.exchange_async(plan.partner)
        elif strategy == "hadpsgd":
            group.ssgd_step(lr, members=list(plan.members), locked=plan.locked)
        else:
            group.locked_update(lr)

    def drain():
        if group is not None:
            group.ack_gate()  # the learner stream waits for the last exchange

    for k in range(args.warmup):
        step(k)
    drain()
    L.check_finite()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for k in range(args.steps):
            step(args.warmup + k)
        drain()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    per_rank_ms = [ms]
    if dist is not None:
        t = torch.zeros(world, device=red_dev)
        t[rank] = ms
        dist.all_reduce(t)  # every rank's device time (straggler analysis); the bench uses the max
        per_rank_ms = [round(float(v), 3) for v in t.tolist()]
        ms = max(per_rank_ms)
        dist.barrier()
    L.check_finite()
    if group is not None:
        group.check()
    frames = args.steps * B * T * world
    value = frames / (ms / 1e3)
    # fwd/bwd kernels + the strategy's sync kernels (sgd+aux / barriers + shard step or mix + aux)
    # per step: ssgd barrier + shard + barrier + aux; adpsgd sender sgd + lock + mix + unlock (receiver
    # lock + sgd + unlock); hadpsgd the group step (+ locks) and the sender's exchange
    sync_launches = {"single": 0, "ssgd": 4 if group is not None else 2, "adpsgd": 4 if group is not None else 2,
                     "hadpsgd": 8}[strategy]  # fused train steps count their SGD launches in kernel_count()
    launches_per_step = L.kernel_count() + sync_launches

    # ---- the sync step alone (NVLink roofline of the sync kernels, SURVEY §8d bytes per unit)
    sync_meas = None
    if group is not None and world > 1:
        reps = 5
        torch.cuda.synchronize()
        dist.barrier()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        P4 = 4 * obj.param_dim
        timed = True
        if strategy in ("ssgd", "hadpsgd"):
            mem = members if strategy == "hadpsgd" else list(range(world))
            lam = len(mem)
            t0e.record(stream)
            for _ in range(reps):
                group.ssgd_step(1e-6, members=mem)
            t1e.record(stream)
            kern = "ds_shard_step between two ds_peer_barrier (whole vector, %d members)" % lam
            rx, tx = (lam - 1) / lam * P4, (lam - 1) / lam * (P4 + P4 // 2)  # gradients in; theta + bf16 snapshot out
        else:
            kern = "ds_pair_mix under the receiver's lock (sender side, whole vector)"
            rx, tx = P4, P4
            if is_sender:
                t0e.record(group.comm)
                for _ in range(reps):
                    group.exchange_async(adpsgd_partner(rank, world, 1))
                t1e.record(group.comm)
                group.ack_gate()
            else:
                timed = False
        torch.cuda.synchronize()
        sms = t0e.elapsed_time(t1e) / reps if timed else 0.0
        t = torch.tensor([sms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sms = float(t.item())
        gbs = max(rx, tx) / (sms * 1e-3) / 1e9 if sms > 0 else None
        sync_meas = {"kernel": kern, "ms": round(sms, 4), "rx_bytes": int(rx), "tx_bytes": int(tx),
                     "achieved_gbs_per_direction": round(gbs, 1) if gbs else None,
                     "peak_gbs_per_direction": 900.0, "peak_kind": "NVLink 5 nominal per direction (spec)",
                     "frac": round(gbs / 900.0, 4) if gbs else None,
                     "path": "same-device IPC (HBM, functional only)" if args.same_device else "NVLink P2P"}

    # ---- end to end through the public Learner API (host indices in, loss out)
    e2e_steps = max(3, min(args.steps, 60))
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    pending = None  # every step's loss is read back; the host issues step k+1 before reading step k's
    for k in range(e2e_steps):
        step(args.warmup + args.steps + k, host=True)
        fut = L.loss_async()
        if pending is not None:
            _ = pending()
        pending = fut
    drain()
    _ = pending()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(e2e_steps * B * T * world / e2e_s, 1), "unit": UNIT, "h2d_bytes_per_step": B * 8,
           "d2h_bytes_per_step": 4}

    # ---- per-phase device times (profiling pass, events around each phase)
    L.set_profile(True)
    L.profile_read()
    nprof = 3
    for k in range(nprof):
        L.gradient_device(idx_dev[k % q], B)
    torch.cuda.synchronize()
    ph = {k: v / nprof for k, v in L.profile_read().items()}
    L.set_profile(False)

    burst, sustained, hbm, peak_kind = _peaks()
    flops_frame = training_flops_per_frame(obj)
    N = B * T
    rec_flops = 2 * obj.layers * 2.0 * N * (8 * 512) * 512  # forward h W_hh^T + backward dh = dG W_hh
    gemm_flops = flops_frame * N - rec_flops
    gemm_tfs = gemm_flops / (ph["gemm"] * 1e-3) / 1e12 if ph["gemm"] > 0 else 0.0
    traffic = None  # DRAM bytes of the same GEMM launches of one step, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "r2f_gemm_traffic.json")) as f:
            tj = json.load(f)
        if B == 256 and obj.layers == 6:
            traffic = {"bytes_per_step": tj["gemm_dram_bytes_per_step"], "launches": tj["gemm_launches_per_step"],
                       "source": "profiles/r2f_gemm_traffic.json (ncu dram__bytes_read+write)"}
    except Exception:
        pass
    gemm_class = {"kernel": "tcgen05 bf16 GEMM-class launches of one step (gemm_kernel + soft-max statistics + "
                            "soft-max/dZ kernels)",
                  "achieved": round(gemm_tfs, 1), "peak": burst, "unit": "TFLOP/s", "frac": round(gemm_tfs / burst, 4),
                  "traffic": traffic, "algorithmic_flop_per_step": gemm_flops}
    # the dominant kernel of the launch list (profiles/r2h_launches.csv: 34.9 %): the BPTT
    # (lstm_bwd3_kernel, the transposed CTA-pair recurrence, one launch per layer)
    bwd_flop = 2.0 * N * (8 * 512) * 512  # dh = dG W_hh, both directions
    bwd_ms = ph["lstm_bwd"] / obj.layers if ph["lstm_bwd"] > 0 else 0.0
    bwd_tfs = bwd_flop / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else 0.0
    bwd_traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2h_kernel_traffic.json")) as f:
            kt = json.load(f)
        if B == 256 and obj.layers == 6 and "lstm_bwd3_kernel" in kt:
            bwd_traffic = kt["lstm_bwd3_kernel"]["dram_bytes_per_launch"]
    except Exception:
        pass
    roof = {"bound": "tensor", "kernel": "lstm_bwd3_kernel (BPTT recurrence + cell backward; latency-bound)",
            "achieved": round(bwd_tfs, 1), "peak": burst, "unit": "TFLOP/s",
            "frac": round(bwd_tfs / burst, 4) if burst else None, "traffic": bwd_traffic,
            "algorithmic_flop_per_launch": bwd_flop, "launch_ms": round(bwd_ms, 4),
            "peak_kind": f"{peak_kind} burst bf16",
            "gemm_class": gemm_class,
            "step_tensor_frac": round(value / world * flops_frame / 1e12 / sustained, 4),
            "step_tensor_frac_peak": f"{peak_kind} sustained bf16 {sustained}",
            "phase_ms": {k: round(v, 3) for k, v in ph.items()}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        fps, sec = cpu_reference(obj, args.batch, 1, 0)
        cpu = {"value": round(fps, 2), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 step of B={args.batch} x 21 frames (the bench config), paper-size model, "
                         "float64 numpy oracle"}
    lib_base = None
    engine_e2e = None
    if rank == 0 and world == 1 and not args.no_library:
        L.close()
        L = None
        lib_base = library_baseline(obj, B)
        engine_e2e = engine_epoch(obj, B, x_host=make_data(obj, args.n_seq, seed=0))

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(obj, B, world, strategy, args, ngroups, gsize),
        "per_rank_ms": per_rank_ms,
        "sync": sync_meas,
        "roofline": roof, "cpu_baseline": cpu, "library_baseline": lib_base, "engine_e2e": engine_e2e, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if group is not None:
        group.close()
    if L is not None:
        L.close()
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without torchrun: launch the N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and relay rank 0's
    line.  Fails loudly when fewer than N GPUs are visible (unless
    --same-device)."""
    import socket

    try:
        import torch

        ndev = torch.cuda.device_count()
    except Exception:  # pragma: no cover
        ndev = 0
    if ndev < args.gpus and not args.same_device:
        print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "error": f"--gpus {args.gpus} but only {ndev} "
                          "CUDA device(s) visible (use --same-device for a functional one-GPU run)"}), flush=True)
        return 2
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--n-seq", type=int, default=16384)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-max-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-library", action="store_true", help="skip the cuDNN/cuBLAS library-path baseline")
    ap.add_argument("--strategy", default="ssgd", choices=["ssgd", "adpsgd", "hadpsgd"])
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on cuda:0 with gloo plumbing (functional check only; p2p transport)")
    ap.add_argument("--adpsgd-mode", default="async", choices=["async", "fused", "lockstep"],
                    help="async: the reference protocol (sender-initiated, ack-gated, receiver lock); fused: "
                         "sender update+mix in one kernel (ds_update_mix); lockstep: pair barriers every step")
    ap.add_argument("--ssgd-mode", default="overlap", choices=["overlap", "after"],
                    help="overlap: each layer's allreduce+SGD runs beside the BPTT of the layers below; after: "
                         "one sharded step after the whole backward")
    ap.add_argument("--straggler-rank", type=int, default=-1, help="rank that sleeps --straggler-sleep s per step")
    ap.add_argument("--straggler-sleep", type=float, default=0.0)
    ap.add_argument("--base-sleep", type=float, default=0.0, help="host sleep per step on every rank (simulated compute)")
    ap.add_argument("--layers", type=int, default=6, help="(tests) smaller models; the bench config is 6")
    ap.add_argument("--classes", type=int, default=32000, help="(tests) smaller output layer; bench config 32000")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # CPU only: rank 0 prints, other ranks (if launched) exit 0
        run_reference_arm(args, rank, max(world, args.gpus))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.warmup < 3:
        args.warmup = 3
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
