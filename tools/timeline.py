"""Per-stream timeline of one fused config-2 training step (B=256): timing
events recorded inside the step graph (DS_TIMELINE=1) after each projection,
recurrence, BPTT, dX / dW GEMM and side-stream SGD, printed as ms from the
step start.  Usage (GPU box):  python tools/timeline.py [steps]"""
import ctypes
import os
import sys

os.environ["DS_TIMELINE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
obj = BlstmObjective()
B, T = 256, obj.frames
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, T, obj.input_dim), dtype=np.float32)
y = rng.integers(0, obj.classes, (2048, T), dtype=np.int64)
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
lib = _lib.load()
lib.ds_debug_timeline.restype = ctypes.c_int
lib.ds_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
for i in range(steps):
    L.train_step(np.arange(B) + (i % 8) * B, 0.1)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16)
_lib.check(lib.ds_debug_timeline(L.handle, buf, len(buf)), "ds_debug_timeline")
prev = {}
for line in buf.value.decode().splitlines():
    name, t = line.split()
    if name == "base_ns":
        continue
    t = float(t)
    print(f"{name:>12s} {t * 1e3:9.1f} us")
