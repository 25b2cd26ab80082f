"""A BPTT launch inside the fused config-2 training step (B=256) against the same kernel alone:
launch start, end of the prologue (W^T in tensor memory), the cell of step 0 (it waits for the
first dY frames when dY streams in from the previous layer's dX), and the per-step period of the
published flags (max over CTAs), next to the step timeline's marks.
Usage (GPU box):  python tools/bptt_insitu.py [layer=3]"""
import ctypes
import os
import sys

os.environ["DS_TIMELINE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

layer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
lib = _lib.load()
obj = BlstmObjective()
B, T = 256, obj.frames
grid = 64
buf = torch.zeros(grid * T * 6 + T * 32 * 2 + 4 * T, device="cuda", dtype=torch.int64)
_lib.check(lib.ds_debug_bptt_trace(ctypes.c_void_p(buf.data_ptr()), layer), "trace")
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, T, obj.input_dim), dtype=np.float32)
y = rng.integers(0, obj.classes, (2048, T), dtype=np.int64)
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
for i in range(6):
    L.train_step(np.arange(B) + (i % 8) * B, 0.1)
torch.cuda.synchronize()
tl = ctypes.create_string_buffer(1 << 16)
lib.ds_debug_timeline.restype = ctypes.c_int
lib.ds_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
_lib.check(lib.ds_debug_timeline(L.handle, tl, len(tl)), "timeline")
marks = {}
for line in tl.value.decode().splitlines():
    n, v = line.split()
    marks[n] = float(v)
base = marks.pop("base_ns")
a = buf.cpu().numpy().astype(np.float64)
m = a[:grid * T * 6].reshape(grid, T, 6)
m = np.where(m > 0, (m - base) / 1e3, np.nan)
print(f"timeline: pre-bptt{layer} {marks[f'pre-bptt{layer}'] * 1e3:.1f}  bptt{layer} {marks[f'bptt{layer}'] * 1e3:.1f} us")
print(f"launch start (min/max over CTAs) {np.nanmin(m[:, 0, 0]):.1f}/{np.nanmax(m[:, 0, 0]):.1f}; "
      f"prologue done {np.nanmin(m[:, 0, 1]):.1f}/{np.nanmax(m[:, 0, 1]):.1f}; "
      f"step-0 cell done (max) {np.nanmax(m[:, 0, 3]):.1f}; step-0 published (max) {np.nanmax(m[:, 0, 4]):.1f} us")
pub = np.nanmax(m[:, :, 4], axis=0)
print("published per step (max over CTAs):", np.round(pub, 1))
print("step periods:", np.round(np.diff(pub), 2), " mean", round(float(np.mean(np.diff(pub))), 2))
