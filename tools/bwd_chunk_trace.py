"""Critical-path decomposition of the split-K BPTT (CTA 0 = dir 0, btile 0,
unit group 0, K slice 0): per chunk j of step s its producer's publish time,
issue and arrival; then MMA done, exchange done, stored, published."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402

B, T, H = 256, 21, 512
N = T * B
lib = _lib.load()
gates = (torch.rand(N, 8 * H, device="cuda")).bfloat16()
cstate = torch.randn(N, 2 * H, device="cuda")
W = (torch.randn(8 * H, H, device="cuda") * 0.05).bfloat16()
WT = torch.cat([W[:4 * H].t(), W[4 * H:].t()], 0).contiguous()
dY = torch.randn(N, 2 * H, device="cuda").bfloat16()
dg = torch.zeros(N, 8 * H, device="cuda", dtype=torch.bfloat16)
counters = torch.zeros(16384, device="cuda", dtype=torch.int32)
grid = 128
tr = torch.zeros(grid * T * 6 + T * 8 * 2, device="cuda", dtype=torch.int64)
s = _lib.stream_ptr()
for i in range(4):
    _lib.check(lib.ds_debug_lstm_bwd(B, T, gates.data_ptr(), cstate.data_ptr(), W.data_ptr(), dY.data_ptr(),
                                     dg.data_ptr(), counters.data_ptr(), tr.data_ptr() if i == 3 else None, s))
torch.cuda.synchronize()
a = tr.cpu().numpy().astype(np.float64)
main = a[:grid * T * 6].reshape(grid, T, 6)
ch = a[grid * T * 6:].reshape(T, 8, 2)
base = a[a > 0].min()
main = np.where(main > 0, main - base, np.nan) / 1e3
ch = np.where(ch > 0, ch - base, np.nan) / 1e3
for st in (6, 10):
    print(f"step {st}")
    for j in range(8):
        c = j  # CTA 0 has ks = 0: chunks 0..7, producer of chunk c is blockIdx c (dir 0, btile 0)
        print(f"  chunk {c}: producer published {main[c, st - 1, 4]:7.2f}  issued {ch[st, j, 0]:7.2f}"
              f"  arrived {ch[st, j, 1]:7.2f}")
    cl = main[0:4, st]
    print("  cluster 0 ctas: mma done", np.round(cl[:, 2], 2), " exchange done", np.round(cl[:, 5], 2),
          " stored", np.round(cl[:, 3], 2), " published", np.round(cl[:, 4], 2))
    print(f"  all ctas: published step {st}: median {np.nanmedian(main[:, st, 4]):.2f} max {np.nanmax(main[:, st, 4]):.2f}")
