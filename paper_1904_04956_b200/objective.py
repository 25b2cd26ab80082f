"""Functional objective API of the reference (objectives.py:23-43,
223-311) for the BLSTM kind, backed by the GPU:

  gradient(obj, w, batch, data)  -> float64 ndarray [param_dim]
  evaluate(obj, w, batch, data)  -> float   (mean CE of the batch)
  heldout_loss(obj, w, data)     -> float   (mean CE of the held-out split)

These are host-array shims (one upload + download per call) kept for
drop-in compatibility and tests; the engines keep weights on the device.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .blstm import BlstmObjective, initial_weights  # noqa: F401  (re-export)


@dataclass(frozen=True)
class Dataset:
    """objectives.py:23-43 with 21-frame sequences as rows: inputs
    [n_seq, T, D] float, targets [n_seq, T] class ids."""

    inputs: np.ndarray
    targets: np.ndarray
    train_indices: np.ndarray
    heldout_indices: np.ndarray

    @property
    def input_dim(self) -> int:
        return self.inputs.shape[-1]

    @property
    def n_train(self) -> int:
        return len(self.train_indices)


def make_blstm_dataset(obj: BlstmObjective, n_seq: int, seed: int) -> Dataset:
    """Synthetic SWB-shaped data: x ~ N(0,1), y ~ U{0..C-1};
    90/10 split as objectives.py:165-171."""
    if n_seq < 10:
        raise ValueError(f"n_samples must be >= 10, got {n_seq}")
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n_seq, obj.frames, obj.input_dim), dtype=np.float32)
    y = rng.integers(0, obj.classes, size=(n_seq, obj.frames), dtype=np.int64)
    n_held = n_seq // 10
    return Dataset(x, y, np.arange(n_seq - n_held), np.arange(n_seq - n_held, n_seq))


_cache: dict = {}
# The reference calls gradient()/evaluate()/heldout_loss() from many learner
# threads at once (RealClock actors, engines/adpsgd.py:138).  The shim keeps one
# cached device learner, so every call holds this lock across its whole
# set_weights -> compute -> read-back sequence: calls serialise (they share one
# GPU stream anyway) and can never read another thread's weights or gradient.
_call_lock = threading.RLock()


def _learner(obj: BlstmObjective, data, batch_len: int):
    from .blstm import DeviceDataset, Learner

    key = (id(obj), id(data))
    ent = _cache.get(key)
    if ent is None or ent[1].max_batch < batch_len:
        dd = DeviceDataset(np.asarray(data.inputs), np.asarray(data.targets))
        mb = max(batch_len, 256)
        ent = (dd, Learner(obj, dd, mb))
        _cache.clear()
        _cache[key] = ent
    return ent[1]


def _check(obj, w):
    if w.ndim != 1 or w.size != obj.param_dim:
        raise ValueError(f"parameter dim mismatch for {obj.kind}: expected {obj.param_dim}, got shape {w.shape}")


def gradient(obj: BlstmObjective, weights: np.ndarray, batch, data) -> np.ndarray:
    _check(obj, weights)
    with _call_lock:
        L = _learner(obj, data, len(batch))
        L.set_weights(weights)
        L.gradient(np.asarray(batch))
        L.check_finite("gradient")
        L.stream.synchronize()
        return L.grad.double().cpu().numpy()


def evaluate(obj: BlstmObjective, weights: np.ndarray, batch, data) -> float:
    _check(obj, weights)
    with _call_lock:
        L = _learner(obj, data, len(batch))
        L.set_weights(weights)
        L.loss(np.asarray(batch))
        val = L.mean_loss()
    if not np.isfinite(val):
        raise ValueError(f"{obj.kind} loss is non-finite (weights diverged?)")
    return val


def heldout_loss(obj: BlstmObjective, weights: np.ndarray, data) -> float:
    _check(obj, weights)
    idx = np.asarray(data.heldout_indices)
    with _call_lock:
        L = _learner(obj, data, min(len(idx), 256))
        L.set_weights(weights)
        return L.heldout_mean(idx)
