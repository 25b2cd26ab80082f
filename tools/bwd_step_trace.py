"""Per-step critical-path marks of the BPTT kernel (B=256, 128 CTAs): median /
max over CTAs of producer flags seen, dG chunks issued, accumulator ready,
partial-dh exchange done, dG stored, flag published.  DS_BWD_IMPL=n traces
the batch-as-N variant."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402

B, T, H = 256, 21, 512
N = T * B
lib = _lib.load()
gates = torch.rand(N, 8 * H, device="cuda").bfloat16()
cstate = torch.randn(N, 2 * H, device="cuda")
W = (torch.randn(8 * H, H, device="cuda") * 0.05).bfloat16()
dY = torch.randn(N, 2 * H, device="cuda").bfloat16()
dg = torch.zeros(N, 8 * H, device="cuda", dtype=torch.bfloat16)
counters = torch.zeros(16384, device="cuda", dtype=torch.int32)
grid = 128 if os.environ.get("DS_BWD") == "1" else 64
tr = torch.zeros(grid * T * 6 + T * 32 * 2 + 4 * T, device="cuda", dtype=torch.int64)
s = _lib.stream_ptr()
for i in range(4):
    _lib.check(lib.ds_debug_lstm_bwd(B, T, gates.data_ptr(), cstate.data_ptr(), W.data_ptr(), dY.data_ptr(),
                                     dg.data_ptr(), counters.data_ptr(), tr.data_ptr() if i == 3 else None, s))
torch.cuda.synchronize()
a = tr.cpu().numpy().astype(np.float64)
main = a[:grid * T * 6].reshape(grid, T, 6)
base = a[a > 0].min()
main = np.where(main > 0, main - base, np.nan) / 1e3
names = ["flags seen", "chunks issued", "acc ready", "exchange done", "dG stored", "published"]
order = [0, 1, 2, 5, 3, 4]
for st in (6, 10, 14):
    med = np.nanmedian(main[:, st, :], axis=0)
    mx = np.nanmax(main[:, st, :], axis=0)
    print(f"step {st}: " + "  ".join(f"{names[i]} {med[k]:.2f}/{mx[k]:.2f}" for i, k in enumerate(order)))
pub = np.nanmax(main[:, :, 4], axis=0)
print("step period (max published):", np.round(np.diff(pub), 2))
ch = a[grid * T * 6:grid * T * 6 + T * 16].reshape(T, 8, 2)
ch = np.where(ch > 0, ch - base, np.nan) / 1e3
for st in (6, 10):
    print(f"cta0 step {st} chunks issued :", np.round(ch[st, :, 0], 2))
    print(f"cta0 step {st} chunks landed :", np.round(ch[st, :, 1], 2))
    print(f"cta0 step {st} marks:", np.round(main[0, st, :], 2))
mm = a[grid * T * 6 + T * 16:grid * T * 6 + T * 18].reshape(T, 2)
mm = np.where(mm > 0, mm - base, np.nan) / 1e3
for st in (6, 10):
    print(f"cta0 step {st} mma issued-last / commit seen by MMA warp:", np.round(mm[st], 2))
cw = a[grid * T * 6 + T * 18:grid * T * 6 + T * 20].reshape(T, 2)
cw = np.where(cw > 0, cw - base, np.nan) / 1e3
for st in (6, 10):
    print(f"cta0 step {st} cell: before / after the staged-input wait:", np.round(cw[st], 2))
