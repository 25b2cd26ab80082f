"""GPU-backed BLSTM objective: the `kind="blstm"` plug-in for the reference's
objective interface (/root/reference/pkg/src/distsgd/objectives.py:223-311).

`BlstmObjective` is the frozen config object the engines carry around
(param_dim / kind / regularization, like TinyMlpObjective at :79-103);
`Learner` owns one learner's device state (fp32 master theta, momentum
velocity, gradient, operand snapshot, libds workspace) and issues the hot
path through the C ABI of include/ds_blstm.h.  There is no CPU fallback: all
compute runs in libds.so on the GPU and any failure raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

HIDDEN = 512  # cells per direction (fixed by the recurrent kernels)
IN_PAD = 272  # layer-0 feature pitch on the device (16-byte TMA rows)


@dataclass(frozen=True)
class BlstmObjective:
    """Paper acoustic model as an objective.  Defaults are the
    paper sizes; smaller configs keep the 512-cell layers (kernel shape)."""

    layers: int = 6
    input_dim: int = 260
    bottleneck: int = 256
    classes: int = 32000
    frames: int = 21
    regularization: float = 0.0

    kind = "blstm"

    def __post_init__(self):
        if self.regularization != 0.0:
            raise ValueError("blstm objective has no L2 term (regularization must be 0)")
        if not 1 <= self.input_dim <= IN_PAD:
            raise ValueError(f"input_dim must be in 1..{IN_PAD}, got {self.input_dim}")
        if self.bottleneck < 64 or self.bottleneck % 64:
            raise ValueError("bottleneck must be a positive multiple of 64")
        if self.classes < 16 or self.classes % 16:
            raise ValueError("classes must be a positive multiple of 16")

    @property
    def param_dim(self) -> int:
        return offsets(self)["total"]

    def cfg(self, max_batch: int) -> _lib.DsCfg:
        return _lib.DsCfg(self.layers, self.input_dim, self.bottleneck, self.classes, self.frames, max_batch)


def offsets(obj: BlstmObjective) -> dict:
    """Flat packing of csrc/layout.h (== oracle/blstm_ref.py BlstmSpec.offsets)."""
    g2 = 8 * HIDDEN
    o = 0
    out = {}
    for l in range(obj.layers):
        d = obj.input_dim if l == 0 else 2 * HIDDEN
        out[("wih", l)] = (o, (g2, d))
        o += g2 * d
        out[("whh", l)] = (o, (g2, HIDDEN))
        o += g2 * HIDDEN
        out[("b", l)] = (o, (g2,))
        o += g2
    out["wb"] = (o, (obj.bottleneck, 2 * HIDDEN))
    o += obj.bottleneck * 2 * HIDDEN
    out["bb"] = (o, (obj.bottleneck,))
    o += obj.bottleneck
    out["wo"] = (o, (obj.classes, obj.bottleneck))
    o += obj.classes * obj.bottleneck
    out["bo"] = (o, (obj.classes,))
    o += obj.classes
    out["total"] = o
    return out


def training_flops_per_frame(obj: BlstmObjective) -> float:
    """Algorithmic training FLOPs per frame: 2*P_w forward, 2*P_w
    weight gradients, 2*(P_w - layer-0 W_ih) input gradients."""
    offs = offsets(obj)
    p_w = 0
    for k, v in offs.items():
        if k == "total":
            continue
        shape = v[1]
        if len(shape) == 2:
            p_w += shape[0] * shape[1]
    w_ih0 = 8 * HIDDEN * obj.input_dim
    return 2.0 * p_w + 2.0 * p_w + 2.0 * (p_w - w_ih0)


def initial_weights(obj: BlstmObjective, seed: int) -> np.ndarray:
    """objectives.py:307-311: 0.1 * N(0, 1) from default_rng((seed, 0))."""
    return 0.1 * np.random.default_rng((seed, 0)).standard_normal(obj.param_dim)


class DeviceDataset:
    """Device-resident copy of a `Dataset` whose inputs are [n_seq, T, D]
    21-frame feature sequences and targets [n_seq, T] class ids
    (objectives.py:23-43 layout, rows = sequences)."""

    def __init__(self, inputs: np.ndarray, targets: np.ndarray, device: int = 0):
        import torch

        if inputs.ndim != 3:
            raise ValueError(f"blstm inputs must be [n_seq, frames, dim], got shape {inputs.shape}")
        n, T, D = inputs.shape
        if targets.shape != (n, T):
            raise ValueError(f"blstm targets must be [n_seq, frames] = {(n, T)}, got {targets.shape}")
        targets = np.asarray(targets)
        if targets.dtype.kind not in "iu":
            if not np.all(np.isfinite(targets)) or not np.all(targets == np.round(targets)):
                raise ValueError("blstm targets must be integer class ids")
        # checked against the objective's class count by Learner (the soft-max
        # kernels never see an out-of-range label)
        self.label_range = (int(targets.min()), int(targets.max())) if targets.size else (0, 0)
        self.n_seq, self.frames, self.input_dim = n, T, D
        self.device = device
        dev = torch.device("cuda", device)
        feats = torch.zeros((n, T, IN_PAD), dtype=torch.bfloat16, device=dev)
        chunk = max(1, (1 << 26) // max(1, T * D))
        for s in range(0, n, chunk):
            part = torch.from_numpy(np.ascontiguousarray(inputs[s:s + chunk], dtype=np.float32))
            feats[s:s + chunk, :, :D] = part.to(dev).to(torch.bfloat16)
        self.feats = feats
        self.labels = torch.from_numpy(np.ascontiguousarray(targets).astype(np.int32)).to(dev)


class Learner:
    """One learner's device state + libds handle (one per GPU, or several
    simulated learners sharing a GPU)."""

    def __init__(self, obj: BlstmObjective, data: DeviceDataset, max_batch: int, device: int = 0,
                 theta0: np.ndarray | None = None, momentum: float = 0.9, stream=None, precision: str = "bf16"):
        import torch

        if data.frames != obj.frames or data.input_dim != obj.input_dim:
            raise ValueError("dataset shape does not match the objective (frames / input_dim)")
        lo, hi = data.label_range
        if lo < 0 or hi >= obj.classes:
            raise ValueError(f"blstm targets must be class ids in [0, {obj.classes}), got range [{lo}, {hi}]")
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be 'bf16' (performance) or 'fp32' (parity), got {precision!r}")
        self.precision = precision
        self.obj = obj
        self.data = data
        self.device = device
        self.max_batch = max_batch
        self.mu = float(momentum)
        lib = _lib.load()
        torch.cuda.set_device(device)
        dev = torch.device("cuda", device)
        h = ctypes.c_void_p()
        cfg = obj.cfg(max_batch)
        _lib.check(lib.ds_blstm_create(ctypes.byref(cfg), device, ctypes.byref(h)), "ds_blstm_create")
        self.handle = h
        if precision == "fp32":
            _lib.check(lib.ds_blstm_set_precision(h, _lib.DS_PREC_FP32), "ds_blstm_set_precision")
        _lib.check(lib.ds_blstm_set_dataset(h, data.feats.data_ptr(), data.labels.data_ptr(), data.n_seq),
                   "ds_blstm_set_dataset")
        P = obj.param_dim
        self.theta = torch.zeros(P, dtype=torch.float32, device=dev)
        self.vel = torch.zeros(P, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(P, dtype=torch.float32, device=dev)
        # the step's loss sum, per index slot (a read-back of one step's loss on the input stream never
        # races the next step); self.loss_sum is the last launched step's
        self._lslot = [torch.zeros(1, dtype=torch.float32, device=dev) for _ in range(2)]
        self.loss_sum = self._lslot[0]
        self._last_slot = -1
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        # minibatch indices: the step reads them from one of two device slots (one cached step graph
        # per slot); a slot is filled on an input stream beside the previous step and the learner stream
        # only waits for that copy's event, so nothing runs between two step graphs on it
        self._islot = [torch.zeros(max_batch, dtype=torch.int64, device=dev) for _ in range(2)]
        self._islot_ready = [torch.cuda.Event() for _ in range(2)]
        self._islot_done = [torch.cuda.Event() for _ in range(2)]  # the step that read the slot has finished
        self._islot_used = [False, False]
        self._islot_i = 0
        self._in_stream = torch.cuda.Stream(device=dev)
        self.idx = self._islot[0]
        # ring of pinned staging buffers: a batch upload only waits for the
        # copy that used the same slot several uploads ago
        self._ring = [torch.zeros(max_batch, dtype=torch.int64).pin_memory() for _ in range(4)]
        self._ring_ptr = [t.data_ptr() for t in self._ring]
        self._ring_ev = [torch.cuda.Event() for _ in range(4)]
        self._ring_used = [False] * 4
        self._ring_i = 0
        self._loss_slots = torch.zeros(4, dtype=torch.float32).pin_memory()
        self._loss_ptr = self._loss_slots.data_ptr()
        self._loss_ev = [torch.cuda.Event() for _ in range(4)]
        self._loss_used = [False] * 4
        self._loss_i = 0
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.batch = 0
        if theta0 is not None:
            self.set_weights(theta0)

    # -- state ----------------------------------------------------------------
    def set_weights(self, w: np.ndarray) -> None:
        import torch

        if w.shape != (self.obj.param_dim,):
            raise ValueError(
                f"parameter dim mismatch for blstm: expected {self.obj.param_dim}, got shape {w.shape}")
        with torch.cuda.stream(self.stream):
            self.theta.copy_(torch.from_numpy(np.asarray(w, dtype=np.float32)).to(self.theta.device))
        self.snapshot()

    def weights(self) -> np.ndarray:
        self.stream.synchronize()
        return self.theta.double().cpu().numpy()

    def snapshot(self) -> None:
        """K2: operand snapshot of the current theta (engines/adpsgd.py:132-134)."""
        lib = _lib.load()
        _lib.check(lib.ds_blstm_cast_snapshot(self.handle, self.theta.data_ptr(), self.stream.cuda_stream),
                   "ds_blstm_cast_snapshot")

    # -- hot path -------------------------------------------------------------
    def _stage(self, fill) -> int:
        """Fill the next index slot on the input stream (`fill(slot_tensor, stream)`), make the learner
        stream wait for it; returns the slot.  Call `_consumed(slot)` after queueing the step."""
        r = self._islot_i
        self._islot_i ^= 1
        if self._islot_used[r]:
            self._in_stream.wait_event(self._islot_done[r])  # the step that read it has run
        fill(self._islot[r], self._in_stream)
        self._islot_ready[r].record(self._in_stream)
        self.stream.wait_event(self._islot_ready[r])
        return r

    def _use_slot(self, r: int) -> None:  # the step about to launch writes its loss into slot r
        self.loss_sum = self._lslot[r]

    def _consumed(self, r: int) -> None:
        self._islot_done[r].record(self.stream)
        self._islot_used[r] = True
        self._last_slot = r

    def _upload_batch(self, batch: np.ndarray):
        """Host indices -> pinned staging ring -> H2D copy into the next device slot.  Returns (B, slot)."""
        B = len(batch)
        if not 1 <= B <= self.max_batch:
            raise ValueError(f"batch of {B} sequences outside 1..{self.max_batch}")
        k = self._ring_i
        self._ring_i = (k + 1) % len(self._ring)
        ev = self._ring_ev[k]
        if self._ring_used[k]:
            ev.synchronize()  # the pinned slot's previous H2D copy has finished
        arr = np.ascontiguousarray(batch, dtype=np.int64)
        ctypes.memmove(self._ring_ptr[k], arr.ctypes.data, B * 8)  # into pinned memory

        def fill(dst, st):
            _lib.check(_lib.load().ds_device_copy(dst.data_ptr(), self._ring_ptr[k], B * 8, st.cuda_stream),
                       "ds_device_copy")
            ev.record(st)

        r = self._stage(fill)
        self._ring_used[k] = True
        return B, r

    def gradient(self, batch: np.ndarray) -> None:
        """gradient(objective, snapshot, batch, dataset) into self.grad
        (objectives.py:236-263); asynchronous on self.stream."""
        B, r = self._upload_batch(batch)
        self.batch = B
        self._use_slot(r)
        lib = _lib.load()
        _lib.check(lib.ds_blstm_fwd_bwd(self.handle, self._islot[r].data_ptr(), B, self.grad.data_ptr(),
                                        self.loss_sum.data_ptr(), self.flag.data_ptr(), self.stream.cuda_stream),
                   "ds_blstm_fwd_bwd")
        self._consumed(r)

    def _stage_device(self, idx_dev, B: int) -> int:
        """Device-resident int64 indices -> the next index slot (a device copy on the input stream,
        after the caller's stream produced them).  Returns the slot."""
        import torch

        if not 1 <= B <= self.max_batch:
            raise ValueError(f"batch of {B} sequences outside 1..{self.max_batch}")
        if idx_dev.dtype != torch.int64 or idx_dev.device != self.theta.device or idx_dev.numel() < B:
            raise ValueError("device indices must be an int64 tensor on the learner's device")
        cur = torch.cuda.current_stream(self.theta.device)

        def fill(dst, st):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                dst[:B].copy_(idx_dev.reshape(-1)[:B], non_blocking=True)
            idx_dev.record_stream(st)

        return self._stage(fill)

    def gradient_device(self, idx_dev, B: int) -> None:
        """Same as `gradient` for indices already resident on the device (never
        synchronises the host)."""
        r = self._stage_device(idx_dev, B)
        self.batch = B
        self._use_slot(r)
        lib = _lib.load()
        _lib.check(lib.ds_blstm_fwd_bwd(self.handle, self._islot[r].data_ptr(), B, self.grad.data_ptr(),
                                        self.loss_sum.data_ptr(), self.flag.data_ptr(), self.stream.cuda_stream),
                   "ds_blstm_fwd_bwd")
        self._consumed(r)

    def train_step(self, batch, lr: float, device_idx: bool = False) -> None:
        """gradient(...) then sgd_step(...) in one fused graph (engines/single.py:
        49-55): each layer's momentum update starts as soon as its gradient is
        final and runs beside the next layer's BPTT.  `batch` is a host index
        array, or (device_idx=True) a device int64 tensor of indices."""
        if lr <= 0:
            raise ValueError(f"learning rate must be > 0, got {lr}")
        if device_idx:
            B = int(batch.shape[0])
            r = self._stage_device(batch, B)
        else:
            B, r = self._upload_batch(batch)
        self.batch = B
        self._use_slot(r)
        lib = _lib.load()
        _lib.check(lib.ds_blstm_train_step(self.handle, self._islot[r].data_ptr(), B, self.theta.data_ptr(),
                                           self.vel.data_ptr(), self.grad.data_ptr(), float(lr), self.mu,
                                           self.loss_sum.data_ptr(), self.flag.data_ptr(), self.stream.cuda_stream),
                   "ds_blstm_train_step")
        self._consumed(r)

    def set_grad_scale(self, frames_total: float) -> None:
        """CE gradient divisor for the next gradients (0 = this batch's frames)."""
        _lib.check(_lib.load().ds_blstm_set_grad_scale(self.handle, float(frames_total)), "ds_blstm_set_grad_scale")

    def set_profile(self, on: bool) -> None:
        _lib.check(_lib.load().ds_blstm_set_profile(self.handle, 1 if on else 0), "ds_blstm_set_profile")

    def profile_read(self) -> dict:
        buf = (ctypes.c_float * 4)()
        _lib.check(_lib.load().ds_blstm_profile_read(self.handle, buf, 4), "ds_blstm_profile_read")
        return {"gemm": buf[0], "lstm_fwd": buf[1], "lstm_bwd": buf[2], "other": buf[3]}

    def kernel_count(self) -> int:
        return int(_lib.load().ds_blstm_kernel_count(self.handle))

    def loss(self, batch: np.ndarray) -> None:
        B, r = self._upload_batch(batch)
        self.batch = B
        self._use_slot(r)
        lib = _lib.load()
        _lib.check(lib.ds_blstm_loss(self.handle, self._islot[r].data_ptr(), B, self.loss_sum.data_ptr(),
                                     self.flag.data_ptr(), self.stream.cuda_stream), "ds_blstm_loss")
        self._consumed(r)

    def heldout_mean(self, idx: np.ndarray) -> float:
        """Mean CE over the sequences `idx` (held-out evaluation,
        objectives.py:286-291), forward only: the per-chunk loss sums are
        accumulated on the device and read back once."""
        import torch

        idx = np.asarray(idx)
        if len(idx) == 0:
            raise ValueError("empty held-out split")
        if getattr(self, "_held_acc", None) is None:
            self._held_acc = torch.zeros(1, dtype=torch.float64, device=self.theta.device)
        acc = self._held_acc
        with torch.cuda.stream(self.stream):
            acc.zero_()
        for s in range(0, len(idx), self.max_batch):
            self.loss(idx[s:s + self.max_batch])
            with torch.cuda.stream(self.stream):
                acc.add_(self.loss_sum)
        self.stream.synchronize()
        return float(acc.item()) / (len(idx) * self.obj.frames)

    def sgd_step(self, lr: float) -> None:
        """sgd_step (optim.py:109-121) fused with the operand snapshot (K9+K2)."""
        if lr <= 0:
            raise ValueError(f"learning rate must be > 0, got {lr}")
        lib = _lib.load()
        _lib.check(lib.ds_sgd_momentum(self.theta.data_ptr(), self.vel.data_ptr(), self.grad.data_ptr(), lr,
                                       self.mu, self.obj.param_dim, self.handle, self.flag.data_ptr(),
                                       self.stream.cuda_stream), "ds_sgd_momentum")

    def check_finite(self, what: str = "gradient") -> None:
        """Raise the reference's ValueError (objectives.py:261-262) when the
        device flagged a non-finite loss / gradient."""
        self.stream.synchronize()
        if int(self.flag.item()) & 1:
            self.flag.zero_()
            raise ValueError(f"blstm {what} is non-finite (weights diverged?)")
        if int(self.flag.item()) & 2:
            self.flag.zero_()
            raise ValueError("minibatch index outside the dataset")
        if int(self.flag.item()) & 4:
            self.flag.zero_()
            raise ValueError("class label outside [0, classes)")
        if int(self.flag.item()) & 8:
            self.flag.zero_()
            raise _lib.DsError("recurrent kernel flag wait timed out (CTAs not co-resident?)")

    def loss_async(self):
        """Queue the read-back of the last step's loss and return a callable that
        waits for that copy and gives the mean CE: the host can issue the next
        step before the loss arrives (pinned 4-slot ring; call each callable
        before issuing four more).  The copy runs on the input stream once the
        step has finished (its loss slot is not reused before the next-but-one
        step), so nothing is queued between two steps on the learner stream."""
        k = self._loss_i
        self._loss_i = (k + 1) % len(self._loss_ev)
        ev = self._loss_ev[k]
        if self._loss_used[k]:
            ev.synchronize()  # the slot's previous copy was consumed
        ptr = self._loss_ptr + 4 * k
        st = self.stream
        if self._last_slot >= 0:
            st = self._in_stream
            st.wait_event(self._islot_done[self._last_slot])
        _lib.check(_lib.load().ds_device_copy(ptr, self.loss_sum.data_ptr(), 4, st.cuda_stream), "ds_device_copy")
        ev.record(st)
        self._loss_used[k] = True
        slots, denom = self._loss_slots, float(self.batch * self.obj.frames)

        def result() -> float:
            ev.synchronize()
            return float(slots[k]) / denom

        return result

    def mean_loss(self) -> float:
        """Mean CE of the last step (waits for self.stream; one pinned 4-byte copy)."""
        out = ctypes.c_float()
        _lib.check(_lib.load().ds_blstm_read_loss(self.handle, self.loss_sum.data_ptr(), self.stream.cuda_stream,
                                                  ctypes.byref(out)), "ds_blstm_read_loss")
        return float(out.value) / (self.batch * self.obj.frames)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.load().ds_blstm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
