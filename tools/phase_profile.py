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
for _ in range(3):
    L.gradient_device(idx, B)
torch.cuda.synchronize()
L.set_profile(True)
L.profile_read()
L.gradient_device(idx, B)
torch.cuda.synchronize()
ms = (ctypes.c_float * 256)()
kinds = (ctypes.c_int32 * 256)()
n = ctypes.c_int32()
_lib.check(_lib.load().ds_blstm_profile_list(L.handle, ms, kinds, 256, ctypes.byref(n)))
names = {0: "gemm", 1: "lstm_fwd", 2: "lstm_bwd", 3: "other"}
tot = 0.0
for i in range(n.value):
    tot += ms[i]
    print(f"{i:3d} {names.get(kinds[i], '?'):9s} {ms[i] * 1e3:9.1f} us")
print(f"total {tot:.3f} ms")
