"""Device half of the learner engines.

`GpuBackend` owns every learner of a run.  Learner i lives on device
`devices[i % len(devices)]` (default: one device) with its own CUDA stream
(`streams="per_learner"`, the default whenever several devices are used) or
all learners share one stream (`streams="single"`, the round-1 layout).

Ordering.  The engines (engines.py) issue operations in the order the
(virtual or real) schedule produces them.  Every operation declares the
learners whose buffers it touches; it waits on the last event of each of
them (cross-stream / cross-device `cudaStreamWaitEvent`) and records a new
one.  So every learner's weights, velocity, gradient and snapshot see
exactly the schedule's sequence of operations — a VirtualClock run replays
the reference's event order bit-identically on any stream / device layout —
while operations on disjoint learners run concurrently.  Gradients on the
same device are additionally chained through a per-device token: the
persistent recurrent kernels need 128 co-resident CTAs and two of them must
never share an SM pool.

Operations map onto the C ABI (include/ds_blstm.h), with peer pointers when
learners sit on different devices (peer access enabled for every pair):

  snapshot  -> ds_blstm_cast_snapshot      (K2; engines/adpsgd.py:132-134)
  gradient  -> ds_blstm_fwd_bwd            (K1,K3-K8; objectives.py:236-263)
  train     -> ds_blstm_train_step         (gradient + sgd_step fused; engines/single.py:53-55)
  sgd_step  -> ds_sgd_momentum (+K2)       (K9; optim.py:109-121)
  mix       -> ds_adpsgd_mix               (K10; engines/adpsgd.py:36-43)
  reduce    -> ds_group_reduce             (K11/K12; collective.py:122-163)
  average   -> ds_average                  (consensus; engines/adpsgd.py:293-295)
  heldout   -> ds_blstm_loss over the held-out split (objectives.py:286-291)
  digest    -> ds_digest                   (debug WeightMessage checksum; engines/common.py:78-104)

The engines are written against this small interface, which is what lets
the CPU test-suite drive the same engine code with a float64 numpy backend
and compare it to the reference engines bit for bit.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .blstm import BlstmObjective, DeviceDataset, Learner


def _ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


class GpuBackend:
    elem_bytes = 4

    def __init__(self, objective: BlstmObjective, dataset, device: int = 0, max_batch: int = 256,
                 precision: str = "bf16", devices: list | None = None, streams: str | None = None):
        import torch

        if not isinstance(objective, BlstmObjective):
            raise ValueError("GpuBackend drives the BLSTM objective (kind='blstm')")
        if not torch.cuda.is_available():
            raise _lib.DsError("GpuBackend needs a CUDA device (there is no CPU fallback)")
        lib = _lib.load()
        self.devices = list(devices) if devices else [device]
        ndev = torch.cuda.device_count()
        if any(d < 0 or d >= ndev for d in self.devices):
            raise ValueError(f"devices {self.devices} outside the {ndev} visible CUDA device(s)")
        streams = streams or ("per_learner" if len(set(self.devices)) > 1 else "single")
        if streams not in ("single", "per_learner"):
            raise ValueError("streams must be 'single' or 'per_learner'")
        if streams == "single" and len(set(self.devices)) > 1:
            raise ValueError("learners on several devices need per-learner streams")
        self.streams = streams
        self.obj = objective
        self.device = self.devices[0]
        self.max_batch = max_batch
        self.precision = precision
        for a in set(self.devices):
            for b in set(self.devices):
                if a != b:
                    _lib.check(lib.ds_enable_peer_access(a, b), "ds_enable_peer_access")
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.Stream(device=torch.device("cuda", self.device))
        self.data = dataset
        self._ddata = {}
        for d in dict.fromkeys(self.devices):
            self._ddata[d] = DeviceDataset(np.asarray(dataset.inputs), np.asarray(dataset.targets), device=d)
        self.ddata = self._ddata[self.device]
        self.heldout = np.asarray(dataset.heldout_indices)
        self.param_dim = objective.param_dim
        self._eval = None
        self._avg = None
        self._digest = None
        self._token = {}  # device -> event of the last gradient issued there
        self.learners: list[Learner] = []

    # -- ordering ---------------------------------------------------------------
    def _run(self, stream, touched, fn, token_device=None):
        """Issue fn() on `stream` after the last operation on every learner in
        `touched` (and on the device's recurrent-kernel token)."""
        import torch

        deps = [L._last_ev for L in touched if getattr(L, "_last_ev", None) is not None]
        if token_device is not None and self._token.get(token_device) is not None:
            deps.append(self._token[token_device])
        for e in deps:
            _wait(stream, e)
        with torch.cuda.device(stream.device), torch.cuda.stream(stream):
            fn()
        ev = torch.cuda.Event()
        ev.record(stream)
        for L in touched:
            L._last_ev = ev
        if token_device is not None:
            self._token[token_device] = ev
        return ev

    # -- learners -----------------------------------------------------------
    def create(self, w0: np.ndarray, momentum: float) -> Learner:
        import torch

        dev = self.devices[len(self.learners) % len(self.devices)]
        stream = self.stream if self.streams == "single" else torch.cuda.Stream(device=torch.device("cuda", dev))
        L = Learner(self.obj, self._ddata[dev], self.max_batch, device=dev, theta0=w0, momentum=momentum,
                    stream=stream, precision=self.precision)
        L._last_ev = None
        self.learners.append(L)
        return L

    def snapshot(self, L: Learner) -> None:
        self._run(L.stream, [L], L.snapshot)

    def gradient(self, L: Learner, batch, frames_total: float = 0.0) -> None:
        def go():
            if frames_total != getattr(L, "_gscale", 0.0):
                L.set_grad_scale(frames_total)
                L._gscale = frames_total
            L.gradient(np.asarray(batch))

        self._run(L.stream, [L], go, token_device=L.device)

    def train_step(self, L: Learner, batch, lr: float) -> None:
        """gradient then sgd_step of one learner (engines/single.py:53-55) as
        the fused device step: each layer's update runs beside the next BPTT
        (bit-identical to gradient + sgd_step, tests/test_gpu_blstm.py)."""
        def go():
            if getattr(L, "_gscale", 0.0):
                L.set_grad_scale(0.0)
                L._gscale = 0.0
            L.train_step(np.asarray(batch), lr)

        self._run(L.stream, [L], go, token_device=L.device)

    def zero_grad(self, L: Learner) -> None:
        self._run(L.stream, [L], L.grad.zero_)

    def sgd_step(self, L: Learner, lr: float) -> None:
        self._run(L.stream, [L], lambda: L.sgd_step(lr))

    def mix(self, a: Learner, b: Learner) -> None:
        self._run(a.stream, [a, b], lambda: _lib.check(_lib.load().ds_adpsgd_mix(
            a.theta.data_ptr(), b.theta.data_ptr(), self.param_dim, a.stream.cuda_stream), "ds_adpsgd_mix"))

    def _group(self, members: list, mode: int, lr: float, chunk_count, divisor: float) -> None:
        """Canonical-order group reduce (one launch per owner rank, each on the
        owner's stream) followed by every member's snapshot refresh."""
        import torch

        lib = _lib.load()
        w = len(members)
        g = _ptr_array([m.grad.data_ptr() for m in members]) if mode == 0 else None
        th = _ptr_array([m.theta.data_ptr() for m in members])
        v = _ptr_array([m.vel.data_ptr() for m in members]) if mode == 0 else None
        chunks = chunk_count or w
        deps = [m._last_ev for m in members if m._last_ev is not None]
        evs = []
        for r, owner in enumerate(members):
            s = owner.stream
            for e in deps:
                _wait(s, e)
            with torch.cuda.device(s.device):
                _lib.check(lib.ds_group_reduce(w, r, g, th, v, None, self.param_dim, chunks, float(lr),
                                               float(members[0].mu) if mode == 0 else 0.0, mode, float(divisor),
                                               s.cuda_stream), "ds_group_reduce")
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        done = _Join(evs)  # every owner's chunks written into every member
        for m in members:
            m._last_ev = done
        for m in members:  # operand snapshot of the new weights
            self._run(m.stream, [m], m.snapshot)

    def group_step(self, members: list, lr: float, chunk_count: int | None = None, divisor: float = 0.0) -> None:
        """SSGD: canonical-order sum of the members' gradients / divisor, then
        every member's momentum update + snapshot (one launch per owner rank)."""
        self._group(members, 0, lr, chunk_count, divisor)

    def group_average(self, members: list, chunk_count: int | None = None) -> None:
        """Hybrid pull: every member's theta <- canonical sum / world."""
        self._group(members, 1, 1.0, chunk_count, 0.0)

    def average(self, members: list):
        """Consensus weights (device tensor on the first device) of the
        members, in member order."""
        import torch

        if self._avg is None:
            with torch.cuda.device(self.device):
                self._avg = torch.empty(self.param_dim, dtype=torch.float32, device=torch.device("cuda", self.device))
        srcs = _ptr_array([m.theta.data_ptr() for m in members])
        holder = _Holder()
        self._run(self.stream, list(members) + [holder], lambda: _lib.check(_lib.load().ds_average(
            len(members), srcs, self._avg.data_ptr(), self.param_dim, self.stream.cuda_stream), "ds_average"))
        self._avg_ev = holder._last_ev
        return self._avg

    # -- debug payload checksum (WeightMessage, engines/common.py:78-104) ----------
    def digest(self, L: Learner) -> str:
        """128-bit device digest of the learner's weights (ds_digest); waits
        for the learner's pending work."""
        import torch

        out = torch.zeros(2, dtype=torch.int64, device=L.theta.device)
        self._run(L.stream, [L], lambda: _lib.check(_lib.load().ds_digest(
            L.theta.data_ptr(), 4 * self.param_dim, out.data_ptr(), L.stream.cuda_stream), "ds_digest"))
        L.stream.synchronize()
        a, b = (int(x) & 0xFFFFFFFFFFFFFFFF for x in out.tolist())
        return f"{a:016x}{b:016x}"

    # -- evaluation -----------------------------------------------------------
    def heldout_loss(self, w) -> float:
        """Mean CE over the held-out split of `w` (a Learner or a device
        tensor), forward only (K13)."""
        import torch

        if self._eval is None:
            self._eval = Learner(self.obj, self.ddata, self.max_batch, device=self.device, stream=self.stream,
                                 precision=self.precision)
            self._eval._last_ev = None
        E = self._eval
        src = w.theta if isinstance(w, Learner) else w
        touched = [E] + ([w] if isinstance(w, Learner) else [])
        if src is self._avg and getattr(self, "_avg_ev", None) is not None:
            self.stream.wait_event(self._avg_ev)

        def go():
            E.theta.copy_(src, non_blocking=True)
            E.snapshot()

        with torch.cuda.stream(self.stream):
            self._run(self.stream, touched, go)
        return E.heldout_mean(self.heldout)

    def weights(self, w) -> np.ndarray:
        import torch

        if isinstance(w, Learner):
            if w._last_ev is not None:
                w._last_ev.synchronize()
            w.stream.synchronize()
            return w.theta.double().cpu().numpy()
        torch.cuda.synchronize(self.device)
        if getattr(self, "_avg_ev", None) is not None:
            self._avg_ev.synchronize()
        return w.double().cpu().numpy()

    def check(self, L: Learner) -> None:
        if L._last_ev is not None:
            L._last_ev.synchronize()
        L.check_finite()

    def sync(self) -> None:
        import torch

        for d in dict.fromkeys(self.devices):
            torch.cuda.synchronize(d)

    def close(self) -> None:
        self.sync()
        for L in self.learners:
            L.close()
        self.learners = []
        if self._eval is not None:
            self._eval.close()
            self._eval = None


def _wait(stream, e) -> None:
    for x in (e.evs if isinstance(e, _Join) else (e,)):
        stream.wait_event(x)


class _Holder:
    """Dependency slot of a buffer that is not a learner (the consensus vector)."""

    _last_ev = None


class _Join:
    """Several events that a later operation must all wait on (member
    refreshes of a group step on different streams)."""

    def __init__(self, evs):
        self.evs = list(evs)

    def synchronize(self):
        for e in self.evs:
            e.synchronize()
