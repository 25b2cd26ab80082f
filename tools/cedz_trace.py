"""Per-tile timeline of the fused soft-max/dZ kernel (softmax_dz.cu) in the
paper-size training step (B=256): for a few CTAs, when MMA1 (logits) and
MMA2 (dZ) of each class tile were issued and when epilogue warp 0 saw the
logits and finished the tile.  Median per-tile deltas tell which stage paces
the loop.

  python tools/cedz_trace.py
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
L.gradient_device(idx, B)
torch.cuda.synchronize()
_lib.check(lib.ds_debug_gemm_trace(buf.data_ptr(), -1))
L.gradient_device(idx, B)
torch.cuda.synchronize()
_lib.check(lib.ds_debug_gemm_trace(None, -1))
L.profile_read()
t = buf.cpu().numpy().reshape(160, 80, 4).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3
ntile = (~np.isnan(t[:, :, 0])).sum(axis=1)
print(f"CTAs traced {int((ntile > 0).sum())}, tiles per CTA (first 80) max {ntile.max()}")
span = np.nanmax(t)
print(f"span of traced tiles {span:.2f} us")
m1 = t[:, :, 0]
m2 = t[:, :, 1]
es = t[:, :, 2]
ee = t[:, :, 3]
print(f"MMA1 issue period median {np.nanmedian(np.diff(m1, axis=1)):.3f} us")
print(f"MMA1 issue -> epilogue sees logits median {np.nanmedian(es - m1):.3f} us")
print(f"epilogue duration (seen -> done) median {np.nanmedian(ee - es):.3f} us")
print(f"epilogue seen -> MMA2 issued median {np.nanmedian(m2 - es):.3f} us")
print(f"MMA2(g) issue -> MMA1(g+1) issue median {np.nanmedian(m1[:, 1:] - m2[:, :-1]):.3f} us")
print(f"epilogue done(g) -> seen(g+1) median {np.nanmedian(es[:, 1:] - ee[:, :-1]):.3f} us")
for c in (0, 1, 77):
    print(f"cta {c}:")
    for g in range(0, 12):
        print(f"  tile {g:2d}: mma1 {t[c, g, 0]:7.2f} epi {t[c, g, 2]:7.2f}-{t[c, g, 3]:7.2f} mma2 {t[c, g, 1]:7.2f}")
