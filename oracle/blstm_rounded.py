"""TEST INFRASTRUCTURE ONLY (never imported by the product path): the float64
oracle of oracle/blstm_ref.py with the device path's rounding points
emulated — every GEMM operand (weights, layer inputs, h, Z, dlogits, dG, dY)
and the stored gate pre-activations rounded to a given mantissa width.

Used to state what a given arithmetic can achieve at BASELINE config 2:
the BF16 perf path is compared with this emulation at 7 bits (so the test
checks the kernels lose nothing beyond BF16 rounding itself), and the FP32
parity mode's bound follows from it at 21-23 bits.  Same packing, same
equations as blstm_ref.loss_and_grad (objectives.py:236-263).
"""

import numpy as np

from . import blstm_ref as O


def rounder(bits):
    """Round float64 -> float32 -> keep `bits` explicit mantissa bits (RNE)."""
    if bits is None:
        return lambda a: a
    drop = 23 - bits

    def r(a):
        f = np.asarray(a, dtype=np.float32)
        u = f.view(np.uint32).astype(np.uint64)
        if drop > 0:
            half = np.uint64(1 << (drop - 1))
            lsb = (u >> np.uint64(drop)) & np.uint64(1)
            u = ((u + half - np.uint64(1) + lsb) >> np.uint64(drop)) << np.uint64(drop)
        return (u.astype(np.uint32).view(np.float32)).astype(np.float64)
    return r


def loss_and_grad_rounded(spec, w, x, y, r):
    """oracle/blstm_ref.loss_and_grad with rounding r() at the device's rounding points."""
    P = O.unpack(spec, w)
    Pr = {k: r(v) for k, v in P.items()}
    B, T, _ = x.shape
    H = spec.hidden
    inp = r(np.ascontiguousarray(np.transpose(x, (1, 0, 2))))
    inputs, acts_all, cs_all = [], [], []
    for l in range(spec.layers):
        proj = r(inp @ Pr[("wih", l)].T + P[("b", l)])  # stored gate pre-activations
        out = np.zeros((T, B, 2 * H))
        acts = np.zeros((T, B, 2, H, 4))
        cs = np.zeros((T, B, 2, H))
        for d in range(2):
            Wd = Pr[("whh", l)][d * 4 * H:(d + 1) * 4 * H]
            h = np.zeros((B, H))
            c = np.zeros((B, H))
            for t in (range(T) if d == 0 else range(T - 1, -1, -1)):
                a = (proj[t, :, d * 4 * H:(d + 1) * 4 * H] + h @ Wd.T).reshape(B, H, 4)
                i, f, o = (O._sigmoid(a[..., k]) for k in (0, 1, 3))
                g = np.tanh(a[..., 2])
                c = f * c + i * g
                h = r(o * np.tanh(c))
                out[t, :, d * H:(d + 1) * H] = h
                acts[t, :, d] = np.stack([i, f, g, o], -1)
                cs[t, :, d] = c
        inputs.append(inp)
        acts_all.append(acts)
        cs_all.append(cs)
        inp = out
    top = inp
    z = r(top @ Pr["wb"].T + P["bb"])
    logits = z @ Pr["wo"].T + P["bo"]
    m = logits.max(-1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(-1, keepdims=True)
    yt = np.ascontiguousarray(y.T).astype(np.int64)
    loss = float(np.mean((m + np.log(s))[..., 0] - np.take_along_axis(logits, yt[..., None], -1)[..., 0]))
    Nf = T * B
    offs = spec.offsets()
    g = np.zeros(spec.param_dim)

    def put(key, arr):
        o, shape = offs[key]
        g[o:o + arr.size] = arr.reshape(-1)

    dlog = e / s
    np.put_along_axis(dlog, yt[..., None], np.take_along_axis(dlog, yt[..., None], -1) - 1.0, -1)
    dlog = r(dlog / Nf)
    put("wo", dlog.reshape(Nf, -1).T @ z.reshape(Nf, -1))
    put("bo", dlog.sum((0, 1)))
    dz = r(dlog @ Pr["wo"])
    put("wb", dz.reshape(Nf, -1).T @ top.reshape(Nf, -1))
    put("bb", dz.sum((0, 1)))
    dy = r(dz @ Pr["wb"])
    for l in range(spec.layers - 1, -1, -1):
        inp, acts, cs = inputs[l], acts_all[l], cs_all[l]
        out_l = inputs[l + 1] if l + 1 < spec.layers else top
        dA = np.zeros((T, B, 8 * H))
        dWhh = np.zeros((8 * H, H))
        for d in range(2):
            Wd = Pr[("whh", l)][d * 4 * H:(d + 1) * 4 * H]
            dh_rec = np.zeros((B, H))
            dcc = np.zeros((B, H))
            for t in (range(T - 1, -1, -1) if d == 0 else range(T)):
                i, f, gg, o = (acts[t, :, d, :, k] for k in range(4))
                c = cs[t, :, d]
                tp = t - 1 if d == 0 else t + 1
                cp = cs[tp, :, d] if 0 <= tp < T else np.zeros_like(c)
                hp = out_l[tp, :, d * H:(d + 1) * H] if 0 <= tp < T else np.zeros((B, H))
                dh = dh_rec + dy[t, :, d * H:(d + 1) * H]
                tc = np.tanh(c)
                dc = dh * o * (1.0 - tc * tc) + dcc
                da = r(np.stack([dc * gg * i * (1.0 - i), dc * cp * f * (1.0 - f), dc * i * (1.0 - gg * gg),
                                 dh * tc * o * (1.0 - o)], -1).reshape(B, 4 * H))
                dcc = dc * f
                dA[t, :, d * 4 * H:(d + 1) * 4 * H] = da
                dWhh[d * 4 * H:(d + 1) * 4 * H] += da.T @ hp
                dh_rec = da @ Wd
        put(("whh", l), dWhh)
        dA2 = dA.reshape(Nf, 8 * H)
        put(("wih", l), dA2.T @ inp.reshape(Nf, -1))
        put(("b", l), dA2.sum(0))
        if l > 0:
            dy = r((dA2 @ Pr[("wih", l)]).reshape(T, B, -1))
    return loss, g
