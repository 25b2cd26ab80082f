"""Per-group timing of the forward recurrence (lstm_fwd2_kernel, B=256: 8 independent groups of 16
CTAs = (direction, 64-row batch block)).  Groups never wait on each other, so the launch lasts as long
as its slowest group: prints each group's step period (its last CTA's publish, step to step) and its
lag behind the fastest group, per launch over several launches, to tell systematic skew (placement)
from noise.

--gemm: a bf16 torch matmul on a second stream, launched right after each recurrence, runs on the
20 SMs the recurrence leaves free (a probe of a projection streaming beside the recurrence)."""
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
s = _lib.stream_ptr()
side = torch.cuda.Stream()
gemm = "--gemm" in sys.argv
Ga = torch.randn(4096, 4096, device="cuda").bfloat16()
Gb = torch.randn(4096, 4096, device="cuda").bfloat16()
for rep in range(8):
    tr = torch.zeros(grid * T * 6 + T * 8 * 2, device="cuda", dtype=torch.int64)
    for i in range(3):
        gates.copy_(G)
        _lib.check(lib.ds_debug_lstm_fwd(B, T, gates.data_ptr(), cstate.data_ptr(), yfull.data_ptr(), W.data_ptr(),
                                         counters.data_ptr(), tr.data_ptr() if i == 2 else None, s))
        if gemm:
            with torch.cuda.stream(side):
                for _ in range(4):
                    Gc = Ga @ Gb
        torch.cuda.synchronize()
    a = tr.cpu().numpy().astype(np.float64)
    main = a[:grid * T * 6].reshape(grid, T, 6)
    pub = main[:, :, 4]  # published (ns, globaltimer)
    base = pub[pub > 0].min()
    pub = (pub - base) / 1e3
    gmax = pub.reshape(8, 16, T).max(axis=1)  # [group, step]
    period = (gmax[:, -1] - gmax[:, 1]) / (T - 2)
    lag = gmax[:, -1] - gmax[:, -1].min()
    print(f"launch {rep}: period/step per group (us) " + " ".join(f"{p:.2f}" for p in period) +
          " | end lag (us) " + " ".join(f"{x:.1f}" for x in lag))
