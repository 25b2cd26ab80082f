"""Critical-path decomposition of the forward recurrence (cluster 0, dir 0,
batch tile 0): for each chunk kb of step s, the latest publish time of its
four producer CTAs, the issue time (multicast TMA) and the arrival at CTA 0."""
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
for st in (6, 10):
    print(f"step {st}")
    for kb in range(8):
        prod = main[4 * kb:4 * kb + 4, st - 1, 4]  # dir 0, btile 0 producers: blockIdx = unit block
        print(f"  chunk {kb}: producers published max {np.nanmax(prod):7.2f} (min {np.nanmin(prod):7.2f})"
              f"  issued {ch[st, kb, 0]:7.2f}  arrived@cta0 {ch[st, kb, 1]:7.2f}")
    print(f"  cta0 mma done {main[0, st, 2]:7.2f}  stored {main[0, st, 3]:7.2f}  published {main[0, st, 4]:7.2f}")
