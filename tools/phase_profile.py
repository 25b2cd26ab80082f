"""Per-launch phase times of one paper-size training step (B=256), from the
CUDA events the profiling mode of libds places between launches."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
obj = BlstmObjective()
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, 21, 260), dtype=np.float32)
y = rng.integers(0, 32000, size=(2048, 21))
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
idx = torch.arange(B, device="cuda")
L.set_profile(True)  # warm-up in the profiling mode too: every launch of the process is a plain one (ncu)
for _ in range(3):
    L.gradient_device(idx, B)
torch.cuda.synchronize()
L.profile_read()
L.gradient_device(idx, B)
torch.cuda.synchronize()
ms = (ctypes.c_float * 256)()
kinds = (ctypes.c_int32 * 256)()
n = ctypes.c_int32()
_lib.check(_lib.load().ds_blstm_profile_list(L.handle, ms, kinds, 256, ctypes.byref(n)))
names = {0: "gemm", 1: "lstm_fwd", 2: "lstm_bwd", 3: "other"}
# algorithmic GFLOP of the GEMM segments in issue order (paper model, N = 21 B)
N = 21 * B
G2, H, LO, BT, C, D0 = 4096, 512, 1024, 256, 32000, 260
gf = [2 * N * G2 * D0] + [2 * N * G2 * LO] * 5 + [2 * N * BT * LO, 2 * N * C * BT, 4 * N * C * BT,
                                                  2 * N * C * BT + 4 * N * BT * LO]  # dW_o + dW_b + dY: one launch
gf += [2 * N * G2 * LO * 2 + 2 * 2 * N * 4 * H * H] * 5 + [2 * N * G2 * D0 + 2 * 2 * N * 4 * H * H]
gi = 0
tot = 0.0
for i in range(n.value):
    tot += ms[i]
    extra = ""
    if kinds[i] == 0 and ms[i] > 0.004 and gi < len(gf):
        extra = f"  {gf[gi] / 1e9:7.1f} GF  {gf[gi] / (ms[i] * 1e-3) / 1e12:7.1f} TF/s"
        gi += 1
    print(f"{i:3d} {names.get(kinds[i], '?'):9s} {ms[i] * 1e3:9.1f} us{extra}")
print(f"total {tot:.3f} ms")
