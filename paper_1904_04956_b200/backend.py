"""Device half of the learner engines.

`GpuBackend` owns every learner of a run on one B200 and ONE CUDA stream:
the engines (engines.py) issue operations in the order the (virtual or real)
schedule produces them, so stream order == schedule order and a
VirtualClock run replays the reference's event order on the GPU exactly.
Operations map onto the C ABI (include/ds_blstm.h):

  snapshot  -> ds_blstm_cast_snapshot      (K2; engines/adpsgd.py:132-134)
  gradient  -> ds_blstm_fwd_bwd            (K1,K3-K8; objectives.py:236-263)
  sgd_step  -> ds_sgd_momentum (+K2)       (K9; optim.py:109-121)
  mix       -> ds_adpsgd_mix               (K10; engines/adpsgd.py:36-43)
  reduce    -> ds_group_reduce             (K11/K12; collective.py:122-163)
  average   -> ds_average                  (consensus; engines/adpsgd.py:293-295)
  heldout   -> ds_blstm_loss over the held-out split (objectives.py:286-291)

The engines are written against this small interface (`create`, `snapshot`,
`gradient`, `sgd_step`, `mix`, `group_step`, `group_average`, `average`,
`heldout_loss`, `weights`, `check`), which is what lets the CPU test-suite
drive the same engine code with a float64 numpy backend and compare it to
the reference engines bit for bit.
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
                 precision: str = "bf16"):
        import torch

        if not isinstance(objective, BlstmObjective):
            raise ValueError("GpuBackend drives the BLSTM objective (kind='blstm')")
        if not torch.cuda.is_available():
            raise _lib.DsError("GpuBackend needs a CUDA device (there is no CPU fallback)")
        _lib.load()
        self.obj = objective
        self.device = device
        self.max_batch = max_batch
        self.precision = precision
        torch.cuda.set_device(device)
        self.stream = torch.cuda.Stream(device=torch.device("cuda", device))
        self.data = dataset
        self.ddata = DeviceDataset(np.asarray(dataset.inputs), np.asarray(dataset.targets), device=device)
        self.heldout = np.asarray(dataset.heldout_indices)
        self.param_dim = objective.param_dim
        self._eval = None
        self._avg = None
        self.learners: list[Learner] = []

    # -- learners -----------------------------------------------------------
    def create(self, w0: np.ndarray, momentum: float) -> Learner:
        L = Learner(self.obj, self.ddata, self.max_batch, device=self.device, theta0=w0, momentum=momentum,
                    stream=self.stream, precision=self.precision)
        self.learners.append(L)
        return L

    def snapshot(self, L: Learner) -> None:
        L.snapshot()

    def gradient(self, L: Learner, batch, frames_total: float = 0.0) -> None:
        if frames_total != getattr(L, "_gscale", 0.0):
            L.set_grad_scale(frames_total)
            L._gscale = frames_total
        L.gradient(np.asarray(batch))

    def train_step(self, L: Learner, batch, lr: float) -> None:
        """gradient then sgd_step of one learner (engines/single.py:53-55) as
        the fused device step: each layer's update runs beside the next BPTT
        (bit-identical to gradient + sgd_step, tests/test_gpu_blstm.py)."""
        if getattr(L, "_gscale", 0.0):
            L.set_grad_scale(0.0)
            L._gscale = 0.0
        L.train_step(np.asarray(batch), lr)

    def zero_grad(self, L: Learner) -> None:
        import torch

        with torch.cuda.stream(self.stream):
            L.grad.zero_()

    def sgd_step(self, L: Learner, lr: float) -> None:
        L.sgd_step(lr)

    def mix(self, a: Learner, b: Learner) -> None:
        _lib.check(_lib.load().ds_adpsgd_mix(a.theta.data_ptr(), b.theta.data_ptr(), self.param_dim,
                                             self.stream.cuda_stream), "ds_adpsgd_mix")

    def group_step(self, members: list, lr: float, chunk_count: int | None = None, divisor: float = 0.0) -> None:
        """SSGD: canonical-order sum of the members' gradients / divisor, then
        every member's momentum update + snapshot (one launch per owner rank)."""
        lib = _lib.load()
        w = len(members)
        g = _ptr_array([m.grad.data_ptr() for m in members])
        th = _ptr_array([m.theta.data_ptr() for m in members])
        v = _ptr_array([m.vel.data_ptr() for m in members])
        chunks = chunk_count or w
        for r in range(w):
            _lib.check(lib.ds_group_reduce(w, r, g, th, v, None, self.param_dim, chunks, float(lr),
                                           float(members[0].mu), 0, float(divisor), self.stream.cuda_stream),
                       "ds_group_reduce")
        for m in members:  # operand snapshot of the new weights (after every owner's chunks)
            m.snapshot()

    def group_average(self, members: list, chunk_count: int | None = None) -> None:
        """Hybrid pull: every member's theta <- canonical sum / world."""
        lib = _lib.load()
        w = len(members)
        th = _ptr_array([m.theta.data_ptr() for m in members])
        chunks = chunk_count or w
        for r in range(w):
            _lib.check(lib.ds_group_reduce(w, r, None, th, None, None, self.param_dim, chunks, 1.0, 0.0, 1, 0.0,
                                           self.stream.cuda_stream), "ds_group_reduce")
        for m in members:
            m.snapshot()

    def average(self, members: list):
        """Consensus weights (device tensor) of the members, in member order."""
        import torch

        if self._avg is None:
            self._avg = torch.empty_like(members[0].theta)
        srcs = _ptr_array([m.theta.data_ptr() for m in members])
        _lib.check(_lib.load().ds_average(len(members), srcs, self._avg.data_ptr(), self.param_dim,
                                          self.stream.cuda_stream), "ds_average")
        return self._avg

    # -- evaluation -----------------------------------------------------------
    def heldout_loss(self, w) -> float:
        """Mean CE over the held-out split of `w` (a Learner or a device
        tensor), forward only (K13)."""
        import torch

        if self._eval is None:
            self._eval = Learner(self.obj, self.ddata, self.max_batch, device=self.device, stream=self.stream,
                                 precision=self.precision)
        E = self._eval
        src = w.theta if isinstance(w, Learner) else w
        with torch.cuda.stream(self.stream):
            E.theta.copy_(src)
        E.snapshot()
        return E.heldout_mean(self.heldout)

    def weights(self, w) -> np.ndarray:
        src = w.theta if isinstance(w, Learner) else w
        self.stream.synchronize()
        return src.double().cpu().numpy()

    def check(self, L: Learner) -> None:
        L.check_finite()

    def sync(self) -> None:
        self.stream.synchronize()

    def close(self) -> None:
        for L in self.learners:
            L.close()
        self.learners = []
        if self._eval is not None:
            self._eval.close()
            self._eval = None
