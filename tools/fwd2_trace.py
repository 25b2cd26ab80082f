"""Critical-path decomposition of the batch-as-N forward recurrence
(lstm_fwd2_kernel, B=256: 128 CTAs).  For CTA 0 (dir 0, batch block 0,
pair 0 leader): per chunk k of step s the issue time (its producer flags
seen) and the arrival (MMA warp saw the full barrier); per step the median
over CTAs of: chunk 0 issued, last chunk issued, accumulator ready,
cell math done, h stored, flag published."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402

B, T, H = 256, 21, 512
N = T * B
lib = _lib.load()
G = (torch.randn(N, 8 * H, device="cuda") * 0.5).bfloat16()
W = (torch.randn(8 * H, H, device="cuda") * 0.05).bfloat16()
gates = G.clone()
cstate = torch.zeros(N, 2 * H, device="cuda")
yfull = torch.zeros((T + 2) * B, 2 * H, device="cuda", dtype=torch.bfloat16)
counters = torch.zeros(16384, device="cuda", dtype=torch.int32)
grid = 128
tr = torch.zeros(grid * T * 6 + T * 8 * 2, device="cuda", dtype=torch.int64)
s = _lib.stream_ptr()
for i in range(4):
    gates.copy_(G)
    _lib.check(lib.ds_debug_lstm_fwd(B, T, gates.data_ptr(), cstate.data_ptr(), yfull.data_ptr(), W.data_ptr(),
                                     counters.data_ptr(), tr.data_ptr() if i == 3 else None, s))
torch.cuda.synchronize()
a = tr.cpu().numpy().astype(np.float64)
main = a[:grid * T * 6].reshape(grid, T, 6)
ch = a[grid * T * 6:].reshape(T, 8, 2)
base = a[a > 0].min()
main = np.where(main > 0, main - base, np.nan) / 1e3
ch = np.where(ch > 0, ch - base, np.nan) / 1e3
names = ["chunk0 issued", "last issued", "acc ready", "cell done", "h stored", "published"]
order = [0, 1, 2, 5, 3, 4]
for st in (6, 10, 14):
    med = np.nanmedian(main[:, st, :], axis=0)
    mx = np.nanmax(main[:, st, :], axis=0)
    print(f"step {st}: " + "  ".join(f"{names[i]} {med[k]:.2f}/{mx[k]:.2f}" for i, k in enumerate(order)))
    print("   cta0 chunks issued :", np.round(ch[st, :, 0], 2))
    print("   cta0 chunks arrived:", np.round(ch[st, :, 1], 2))
pub = np.nanmax(main[:, :, 4], axis=0)
print("step period (max published):", np.round(np.diff(pub), 2))
