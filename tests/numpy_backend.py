"""TEST INFRASTRUCTURE: a float64 numpy backend for the engines in
paper_1904_04956_b200/engines.py.  It performs the reference's own arithmetic
(sgd_step optim.py:109-121, adpsgd_mix adpsgd.py:36-43, canonical ring
allreduce collective.py:122-163, np.mean consensus adpsgd.py:293-295) with
an injected `gradient` / `heldout_loss`, so the engine + runtime restatement
can be compared with the reference engines bit for bit on CPU.  Never used
by the product path (which is GpuBackend, CUDA only)."""

from __future__ import annotations

import numpy as np


class _L:
    def __init__(self, w, mu):
        self.w = np.array(w, dtype=np.float64, copy=True)
        self.v = np.zeros_like(self.w)
        self.mu = mu
        self.snap = self.w.copy()
        self.g = None


class NumpyBackend:
    elem_bytes = 8

    def __init__(self, objective, dataset, gradient_fn, heldout_fn, chunk_count=None):
        self.obj = objective
        self.data = dataset
        self.grad_fn = gradient_fn
        self.heldout_fn = heldout_fn
        self.param_dim = objective.param_dim

    def create(self, w0, momentum):
        return _L(w0, momentum)

    def snapshot(self, L):
        L.snap = L.w.copy()

    def gradient(self, L, batch, frames_total: float = 0.0):
        g = self.grad_fn(self.obj, L.snap, batch, self.data)
        if frames_total:  # member of an H-ADPSGD group: frame-weighted share of the union batch
            x = self.data.inputs
            per = x.shape[1] if x.ndim == 3 else 1
            g = g * (len(batch) * per / frames_total)
        L.g = g

    def train_step(self, L, batch, lr):
        self.gradient(L, batch)
        self.sgd_step(L, lr)

    def zero_grad(self, L):
        L.g = np.zeros(self.param_dim)

    def _step(self, L, g, lr):
        L.v *= L.mu
        L.v += g
        L.w = L.w - lr * L.v
        L.snap = L.w.copy()

    def sgd_step(self, L, lr):
        self._step(L, L.g, lr)

    def mix(self, a, b):
        m = (a.w + b.w) / 2.0
        a.w = m
        b.w = m.copy()

    def _ring_sum(self, vecs, chunk_count):
        w = len(vecs)
        c = chunk_count or w
        dim = len(vecs[0])
        size = -(-dim // c)
        out = np.empty(dim)
        for j in range(c):
            lo, hi = min(j * size, dim), min((j + 1) * size, dim)
            o = j % w
            s = vecs[o][lo:hi].astype(np.float64).copy()
            for k in range(1, w):
                s = s + vecs[(o + k) % w][lo:hi]
            out[lo:hi] = s
        return out

    def group_step(self, members, lr, chunk_count=None, divisor=0.0):
        tot = self._ring_sum([m.g for m in members], chunk_count)
        g = tot / (divisor if divisor > 0 else len(members))
        for m in members:
            self._step(m, g, lr)

    def group_average(self, members, chunk_count=None):
        tot = self._ring_sum([m.w for m in members], chunk_count)
        avg = tot / len(members)
        for m in members:
            m.w = avg.copy()
            m.snap = m.w.copy()

    def average(self, members):
        return np.mean(np.stack([m.w for m in members]), axis=0)

    def digest(self, L):
        import hashlib

        return hashlib.blake2b(np.ascontiguousarray(L.w).tobytes(), digest_size=16).hexdigest()

    def heldout_loss(self, w):
        return self.heldout_fn(self.obj, w.w if isinstance(w, _L) else w, self.data)

    def weights(self, w):
        return (w.w if isinstance(w, _L) else w).copy()

    def check(self, L):
        if L.g is not None and not np.all(np.isfinite(L.g)):
            raise ValueError(f"{self.obj.kind} gradient is non-finite (weights diverged?)")

    def sync(self):
        pass
