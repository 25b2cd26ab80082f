"""CPU oracle (TEST INFRASTRUCTURE ONLY — never imported by the product path).

A float64 numpy restatement of the paper's acoustic model (PAPER.md:202:
6 bidirectional LSTM layers of 1024 cells = 512 per direction, a 256-unit
linear bottleneck, a 32000-way soft-max, 21 unrolled frames of 260-dim
features) as an objective of the reference's `objectives.py` kind:
    loss  = mean over all B*T frames of cross-entropy   (cf. evaluate, :223-233)
    grad  = exact analytic gradient of that loss         (cf. gradient, :236-263)
    theta = one flat float64 vector                       (cf. :3-5, :97-103)
The BLSTM is NOT in the reference, so this module is a new
restatement; it is pinned by (a) the reference's own central-difference
oracle `finite_diff_gradient` (objectives.py:266-283) on a coordinate subset
and (b) torch.nn.LSTM in float64 (tests/test_oracle.py).  Parity status:
schedule/sync pinned to the reference itself; BLSTM math pinned by FD +
torch cross-check ("parity unpinned by the reference" for the model math,
see DESIGN.md §Oracle).

Flat packing (identical to paper_1904_04956_b200/csrc/layout.h):
  for each layer l:  W_ih[l] [2*4H, D_l], W_hh[l] [2*4H, H], b[l] [2*4H]
                     rows = dir*4H + unit*4 + gate, gate order (i, f, g, o)
  then W_b [Bn, 2H], b_b [Bn] (omitted when Bn == 0), W_o [C, Bn or 2H], b_o [C]
Single bias per gate row, zero initial (h, c) for every 21-frame subsequence.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class BlstmSpec:
    layers: int = 6
    input_dim: int = 260
    hidden: int = 512  # cells per direction
    bottleneck: int = 256  # 0 = no bottleneck (tiny config)
    classes: int = 32000
    frames: int = 21

    def in_dim(self, l: int) -> int:
        return self.input_dim if l == 0 else 2 * self.hidden

    @property
    def top_dim(self) -> int:
        return self.bottleneck if self.bottleneck else 2 * self.hidden

    def offsets(self) -> dict:
        H4 = 8 * self.hidden
        o = 0
        offs = {}
        for l in range(self.layers):
            offs[("wih", l)] = (o, (H4, self.in_dim(l)))
            o += H4 * self.in_dim(l)
            offs[("whh", l)] = (o, (H4, self.hidden))
            o += H4 * self.hidden
            offs[("b", l)] = (o, (H4,))
            o += H4
        if self.bottleneck:
            offs["wb"] = (o, (self.bottleneck, 2 * self.hidden))
            o += self.bottleneck * 2 * self.hidden
            offs["bb"] = (o, (self.bottleneck,))
            o += self.bottleneck
        offs["wo"] = (o, (self.classes, self.top_dim))
        o += self.classes * self.top_dim
        offs["bo"] = (o, (self.classes,))
        o += self.classes
        offs["total"] = o
        return offs

    @property
    def param_dim(self) -> int:
        return self.offsets()["total"]


PAPER = BlstmSpec()
TINY = BlstmSpec(layers=2, input_dim=260, hidden=32, bottleneck=0, classes=32, frames=21)


def unpack(spec: BlstmSpec, w: np.ndarray) -> dict:
    offs = spec.offsets()
    out = {}
    for k, v in offs.items():
        if k == "total":
            continue
        o, shape = v
        out[k] = w[o:o + int(np.prod(shape))].reshape(shape)
    return out


def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def _check(spec: BlstmSpec, w: np.ndarray) -> None:
    # error text of objectives.py:186-191
    if w.ndim != 1 or w.size != spec.param_dim:
        raise ValueError(f"parameter dim mismatch for blstm: expected {spec.param_dim}, got shape {w.shape}")


def forward(spec: BlstmSpec, w: np.ndarray, x: np.ndarray, y: np.ndarray, keep: bool = False):
    """x: [B, T, D] float, y: [B, T] int. Returns (mean CE, cache)."""
    _check(spec, w)
    P = unpack(spec, w)
    B, T, _ = x.shape
    H = spec.hidden
    inp = np.ascontiguousarray(np.transpose(x, (1, 0, 2)), dtype=np.float64)  # [T, B, D]
    cache = {"inputs": [], "acts": [], "cs": [], "outs": []}
    for l in range(spec.layers):
        Wih, Whh, b = P[("wih", l)], P[("whh", l)], P[("b", l)]
        out = np.zeros((T, B, 2 * H))
        acts_l = np.zeros((T, B, 2, H, 4))
        cs_l = np.zeros((T, B, 2, H))
        proj = inp @ Wih.T + b  # [T, B, 8H]
        for d in range(2):
            Wd = Whh[d * 4 * H:(d + 1) * 4 * H]
            h = np.zeros((B, H))
            c = np.zeros((B, H))
            order = range(T) if d == 0 else range(T - 1, -1, -1)
            for t in order:
                a = (proj[t, :, d * 4 * H:(d + 1) * 4 * H] + h @ Wd.T).reshape(B, H, 4)
                i = _sigmoid(a[..., 0])
                f = _sigmoid(a[..., 1])
                g = np.tanh(a[..., 2])
                o = _sigmoid(a[..., 3])
                c = f * c + i * g
                h = o * np.tanh(c)
                out[t, :, d * H:(d + 1) * H] = h
                acts_l[t, :, d] = np.stack([i, f, g, o], -1)
                cs_l[t, :, d] = c
        cache["inputs"].append(inp)
        cache["acts"].append(acts_l)
        cache["cs"].append(cs_l)
        inp = out
    cache["top_in"] = inp
    if spec.bottleneck:
        z = inp @ P["wb"].T + P["bb"]
    else:
        z = inp
    cache["z"] = z
    logits = z @ P["wo"].T + P["bo"]  # [T, B, C]
    m = logits.max(-1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(-1, keepdims=True)
    lse = (m + np.log(s))[..., 0]
    yt = np.ascontiguousarray(y.T).astype(np.int64)  # [T, B]
    tgt = np.take_along_axis(logits, yt[..., None], -1)[..., 0]
    loss = float(np.mean(lse - tgt))
    if keep:
        cache["prob"] = e / s
        cache["yt"] = yt
        cache["P"] = P
    return loss, cache


def loss(spec: BlstmSpec, w: np.ndarray, x: np.ndarray, y: np.ndarray) -> float:
    val, _ = forward(spec, w, x, y)
    if not np.isfinite(val):
        raise ValueError("blstm loss is non-finite (weights diverged?)")
    return val


def loss_and_grad(spec: BlstmSpec, w: np.ndarray, x: np.ndarray, y: np.ndarray):
    val, cache = forward(spec, w, x, y, keep=True)
    P = cache["P"]
    T, B, C = cache["prob"].shape
    H = spec.hidden
    Nf = T * B
    offs = spec.offsets()
    g = np.zeros(spec.param_dim)

    def put(key, arr):
        o, shape = offs[key]
        g[o:o + arr.size] = arr.reshape(-1)

    dlog = cache["prob"].copy()
    np.put_along_axis(dlog, cache["yt"][..., None], np.take_along_axis(dlog, cache["yt"][..., None], -1) - 1.0, -1)
    dlog /= Nf
    z = cache["z"]
    put("wo", dlog.reshape(Nf, -1).T @ z.reshape(Nf, -1))
    put("bo", dlog.sum((0, 1)))
    dz = dlog @ P["wo"]
    if spec.bottleneck:
        top = cache["top_in"]
        put("wb", dz.reshape(Nf, -1).T @ top.reshape(Nf, -1))
        put("bb", dz.sum((0, 1)))
        dy = dz @ P["wb"]
    else:
        dy = dz
    for l in range(spec.layers - 1, -1, -1):
        inp = cache["inputs"][l]
        acts = cache["acts"][l]
        cs = cache["cs"][l]
        Whh = P[("whh", l)]
        dA = np.zeros((T, B, 8 * H))
        dWhh = np.zeros_like(Whh)
        for d in range(2):
            Wd = Whh[d * 4 * H:(d + 1) * 4 * H]
            dh_rec = np.zeros((B, H))
            dcc = np.zeros((B, H))
            order = range(T - 1, -1, -1) if d == 0 else range(T)
            # h_prev (forward order) for dW_hh
            out_l = cache["inputs"][l + 1] if l + 1 < spec.layers else cache["top_in"]
            for t in order:
                i, f, gg, o = (acts[t, :, d, :, k] for k in range(4))
                c = cs[t, :, d]
                tp = t - 1 if d == 0 else t + 1
                cp = cs[tp, :, d] if 0 <= tp < T else np.zeros_like(c)
                hp = out_l[tp, :, d * H:(d + 1) * H] if 0 <= tp < T else np.zeros((B, H))
                dh = dh_rec + dy[t, :, d * H:(d + 1) * H]
                tc = np.tanh(c)
                dc = dh * o * (1.0 - tc * tc) + dcc
                da = np.stack([dc * gg * i * (1.0 - i), dc * cp * f * (1.0 - f), dc * i * (1.0 - gg * gg),
                               dh * tc * o * (1.0 - o)], -1).reshape(B, 4 * H)
                dcc = dc * f
                dA[t, :, d * 4 * H:(d + 1) * 4 * H] = da
                dWhh[d * 4 * H:(d + 1) * 4 * H] += da.T @ hp
                dh_rec = da @ Wd
        put(("whh", l), dWhh)
        dA2 = dA.reshape(Nf, 8 * H)
        put(("wih", l), dA2.T @ inp.reshape(Nf, -1))
        put(("b", l), dA2.sum(0))
        if l > 0:
            dy = (dA2 @ P[("wih", l)]).reshape(T, B, -1)
    if not np.isfinite(val) or not np.all(np.isfinite(g)):
        raise ValueError("blstm gradient is non-finite (weights diverged?)")
    return val, g


def initial_weights(spec: BlstmSpec, seed: int) -> np.ndarray:
    """objectives.py:307-311: 0.1 * N(0, 1) from default_rng((seed, 0))."""
    rng = np.random.default_rng((seed, 0))
    return 0.1 * rng.standard_normal(spec.param_dim)


def make_dataset(spec: BlstmSpec, n_seq: int, seed: int):
    """Synthetic SWB-shaped data: x ~ N(0,1) [n_seq, T, D],
    y ~ U{0..C-1} [n_seq, T]; 90/10 split as objectives.py:165-171."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n_seq, spec.frames, spec.input_dim))
    y = rng.integers(0, spec.classes, size=(n_seq, spec.frames))
    n_held = n_seq // 10
    n_train = n_seq - n_held
    return x, y, np.arange(n_train), np.arange(n_train, n_seq)
