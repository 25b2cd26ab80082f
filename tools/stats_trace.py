"""Per-tile timeline of the soft-max statistics kernel (softmax_dz.cu,
ce_stats_kernel) in the paper-size step: MMA1 issue, W-stage refill issue,
epilogue warp 0 logits seen / tile done.  Same switch as tools/cedz_trace.py
(both fused output-layer kernels record while it is set; the statistics
kernel runs first, so the buffer is read after a loss-only step).

  python tools/stats_trace.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

B = 256
lib = _lib.load()
obj = BlstmObjective()
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, 21, 260), dtype=np.float32)
y = rng.integers(0, 32000, size=(2048, 21))
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
idx = torch.arange(B, device="cuda")
for _ in range(3):
    L.gradient_device(idx, B)
torch.cuda.synchronize()
L.set_profile(True)
buf = torch.zeros(160 * 80 * 4, dtype=torch.int64, device="cuda")
_lib.check(lib.ds_debug_gemm_trace(buf.data_ptr(), -1))
L.loss(np.arange(B))  # loss only: the gradient kernel would overwrite the record
torch.cuda.synchronize()
_lib.check(lib.ds_debug_gemm_trace(None, -1))
L.profile_read()
t = buf.cpu().numpy().reshape(160, 80, 4).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3
m1, wl, es, ee = t[:, :, 0], t[:, :, 1], t[:, :, 2], t[:, :, 3]
print(f"MMA1 issue period median {np.nanmedian(np.diff(m1, axis=1)):.3f} us")
print(f"W refill issue period median {np.nanmedian(np.diff(wl, axis=1)):.3f} us")
print(f"W refill issued -> MMA1 of that tile {np.nanmedian(m1 - wl):.3f} us")
print(f"MMA1 issue -> epilogue sees logits {np.nanmedian(es - m1):.3f} us")
print(f"epilogue tile (seen -> done) {np.nanmedian(ee - es):.3f} us; done(g) -> seen(g+1) "
      f"{np.nanmedian(es[:, 1:] - ee[:, :-1]):.3f} us")
for c in (0, 77):
    print(f"cta {c}:")
    for g in range(12):
        print(f"  tile {g:2d}: wload {t[c, g, 1]:7.2f} mma1 {t[c, g, 0]:7.2f} epi {t[c, g, 2]:7.2f}-{t[c, g, 3]:7.2f}")
