"""Time one bidirectional layer's recurrent forward/backward kernels at the
paper shape and print per-step phase marks from the in-kernel globaltimer
trace (producer ready / loads issued / MMA done / step published)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
T = 21
H = 512
N = T * B
lib = _lib.load()
dev = "cuda"
G = (torch.randn(N, 8 * H, device=dev) * 0.5).bfloat16()
W = (torch.randn(8 * H, H, device=dev) * 0.05).bfloat16()
WT = torch.cat([W[:4 * H].t(), W[4 * H:].t()], 0).contiguous()
gates = G.clone()
cstate = torch.zeros(N, 2 * H, device=dev)
yfull = torch.zeros((T + 2) * B, 2 * H, device=dev, dtype=torch.bfloat16)
counters = torch.zeros(16384, device=dev, dtype=torch.int32)
dY = torch.randn(N, 2 * H, device=dev).bfloat16()
dg = torch.zeros(N, 8 * H, device=dev, dtype=torch.bfloat16)
ntile = (B + 127) // 128
grid = 64 * ntile
trace = torch.zeros(grid * T * 6 + T * 32 * 2, device=dev, dtype=torch.int64)
s = _lib.stream_ptr()


def fwd(tr=None):
    _lib.check(lib.ds_debug_lstm_fwd(B, T, gates.data_ptr(), cstate.data_ptr(), yfull.data_ptr(), W.data_ptr(),
                                     counters.data_ptr(), tr, s))


def bwd(tr=None):
    _lib.check(lib.ds_debug_lstm_bwd(B, T, gates.data_ptr(), cstate.data_ptr(), W.data_ptr(), dY.data_ptr(),
                                     dg.data_ptr(), counters.data_ptr(), tr, s))


ref_out = {}
for name, fn in (("fwd", fwd), ("bwd", bwd)):
    for _ in range(3):
        gates.copy_(G)
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch ({e0.elapsed_time(e1) / 10 * 1e3 / T:.2f} us/step)")
    trace.zero_()
    fn(trace.data_ptr())
    torch.cuda.synchronize()
    full = trace.cpu().numpy().astype(np.float64)
    g = grid
    tr = full[:g * T * 6].reshape(g, T, 6)
    t2 = full[g * T * 6:g * T * 6 + T * 64].reshape(T, 32, 2)
    base = tr[tr > 0].min()
    tr = np.where(tr > 0, tr - base, np.nan) / 1e3
    # per step: median over CTAs of (ready, issued, mma_done, published)
    for st in range(0, T, 4):
        med = np.nanmedian(tr[:, st, :], axis=0)
        mx = np.nanmax(tr[:, st, :], axis=0)
        print(f"  step {st:2d} med ready {med[0]:7.2f} issued {med[1]:7.2f} mma {med[2]:7.2f} stored {med[3]:7.2f}"
              f" lastwarp {med[5]:7.2f} pub {med[4]:7.2f} | max pub {mx[4]:7.2f}")
    pub = np.nanmax(tr[:, :, 4], axis=0)
    late = np.argsort(-np.nan_to_num(tr[:, 8, 4]))[:6]
    print("  slowest CTAs at step 8:", [(int(c), round(float(tr[c, 8, 4]), 1)) for c in late],
          "first-step ready of those:", [round(float(np.nanmin(tr[c, :, 0])), 1) for c in late])
    if False:
        b2 = np.where(t2 > 0, t2 - base, np.nan) / 1e3
        for st in (5, 6):
            print("  cta0 step", st, "stage-ready:", np.round(b2[st, :, 0], 2))
            print("  cta0 step", st, "flag-ok   :", np.round(b2[st, :, 1], 2))
    print("  step period (max published):", np.round(np.diff(pub), 2))

    ref_out[name] = (yfull.clone(), dg.clone())
import os
print("checksums", float(yfull.float().abs().sum()), float(dg.float().abs().sum()))
