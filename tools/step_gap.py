"""Device time between consecutive fused training steps (config 2, B=256) outside the step graph:
CUDA events recorded on the learner stream around every step give the period; the in-graph stamps
(DS_TIMELINE=1) give the span from the graph's first to its last node.  Variants: the index copy
into the learner buffer per step (Learner.train_step(device_idx=True)) vs the library call alone."""
import ctypes
import os
import sys

TL = "--no-timeline" not in sys.argv
if TL:
    os.environ["DS_TIMELINE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

obj = BlstmObjective()
B, T = 256, obj.frames
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, T, obj.input_dim), dtype=np.float32)
y = rng.integers(0, obj.classes, (2048, T), dtype=np.int64)
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
lib = _lib.load()
lib.ds_debug_timeline.restype = ctypes.c_int
lib.ds_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
dev = [torch.from_numpy(rng.permutation(2048)[:B]).cuda() for _ in range(8)]
for k in range(8):
    L.train_step(dev[k], 0.01, device_idx=True)
torch.cuda.synchronize()


def direct(k, ptr=None):  # the C ABI call alone
    _lib.check(lib.ds_blstm_train_step(L.handle, ptr or L.idx.data_ptr(), B, L.theta.data_ptr(), L.vel.data_ptr(),
                                       L.grad.data_ptr(), ctypes.c_float(0.01), ctypes.c_float(L.mu),
                                       L.loss_sum.data_ptr(), L.flag.data_ptr(), L.stream.cuda_stream), "step")


for name, fn in (("train_step(device_idx)", lambda k: L.train_step(dev[k % 8], 0.01, device_idx=True)),
                 ("  ..current stream default", None),
                 ("train_step(same tensor)", lambda k: L.train_step(dev[0], 0.01, device_idx=True)),
                 ("ABI, one index buffer", direct),
                 ("ABI, 8 index buffers", lambda k: direct(k, dev[k % 8].data_ptr()))):
    n = 40
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    if fn is None:  # the bench's call: indices produced before the loop, caller on the default stream
        for k in range(n):
            ev[k].record(L.stream)
            L.train_step(dev[k % 8], 0.01, device_idx=True)
        ev[n].record(L.stream)
    else:
        with torch.cuda.stream(L.stream):  # the caller's stream is the learner's: the index copy waits for
            for k in range(n):             # the previous step (wait_stream), serialising it behind it
                ev[k].record(L.stream)
                fn(k)
            ev[n].record(L.stream)
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(n)]
    if not TL:
        print(f"{name:26s}: period median {np.median(per[5:]):8.1f} us")
        continue
    buf = ctypes.create_string_buffer(1 << 16)
    _lib.check(lib.ds_debug_timeline(L.handle, buf, len(buf)), "timeline")
    marks = {}
    for line in buf.value.decode().splitlines():
        a, b = line.split()
        marks[a] = float(b)
    span = marks["end"] * 1e3
    print(f"{name:26s}: period median {np.median(per[5:]):8.1f} us, in-graph start->end {span:8.1f} us, "
          f"outside {np.median(per[5:]) - span:6.1f} us")
