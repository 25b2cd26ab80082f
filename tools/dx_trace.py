"""Unit timeline of the streamed dX GEMM of one layer inside the fused
config-2 training step (B=256): per CTA pair, every unit's tile index, when
its producer started waiting for the BPTT gate and when the gate passed, when
the MMA issuer started / finished it and when its epilogue ended, in us from
the step start, next to the step timeline (DS_TIMELINE marks).
Usage (GPU box):  python tools/dx_trace.py [layer=3]   (layer 0: the late layer-0 weight gradients)"""
import ctypes
import os
import sys

os.environ["DS_TIMELINE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

TILES, FIELDS = 32, 11
layer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
lib = _lib.load()
buf = torch.zeros(160 * TILES * FIELDS, dtype=torch.int64, device="cuda")
_lib.check(lib.ds_debug_gemm_trace(ctypes.c_void_p(buf.data_ptr()), -2 - layer), "trace")
obj = BlstmObjective()
B, T = 256, obj.frames
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
for n in (f"pre-bptt{layer}", f"bptt{layer}", f"dX{layer}", f"pre-bptt{layer - 1}", f"bptt{layer - 1}", "dW0-early",
          "grp0", "sgd-main", "end"):
    if n in marks:
        print(f"{n:>12s} {marks[n] * 1e3:8.1f} us")
t = buf.cpu().numpy().reshape(160, TILES, FIELDS).astype(np.float64)
lead = t[0::2]
rel = lambda v: np.where(v > 0, (v - base) / 1e3, np.nan)  # noqa: E731
print("pair: unit (gate wait -> pass | mma start -> end | epi end) ...")
busy = []
for p in range(lead.shape[0]):
    if lead[p, 0, 7] == 0:
        continue
    row = []
    for u in range(TILES):
        if lead[p, u, 0] == 0:
            break
        g0, g1 = rel(lead[p, u, 8]), rel(lead[p, u, 9])
        m0, m1, e1 = rel(lead[p, u, 0]), rel(lead[p, u, 2]), rel(lead[p, u, 4])
        busy.append(m1 - m0)
        row.append(f"[{g0:6.1f}>{g1:6.1f}|{m0:6.1f}-{m1:6.1f}|{e1:6.1f}]")
    print(f"{p:3d}: " + " ".join(row))
print("mean MMA span per unit %.2f us over %d units" % (np.nanmean(busy), len(busy)))
es, ee, rd = rel(lead[:, :, 3]), rel(lead[:, :, 4]), rel(lead[:, :, 10])
print("epilogue (mean / max us): %.2f / %.2f, start -> output counted %.2f / %.2f" % (
    np.nanmean(ee - es), np.nanmax(ee - es), np.nanmean(rd - es), np.nanmax(rd - es)))
print("epilogue start - MMA end (mean / max us): %.2f / %.2f" % (np.nanmean(es - rel(lead[:, :, 2])), np.nanmax(es - rel(lead[:, :, 2]))))
ms, me = rel(lead[:, :, 0]), rel(lead[:, :, 4])
print("launch: first MMA %.1f us, last epilogue %.1f us; CTA starts %.1f .. %.1f us" % (
    np.nanmin(ms), np.nanmax(me), np.nanmin(rel(t[:, 0, 7])), np.nanmax(rel(t[:, 0, 7]))))
