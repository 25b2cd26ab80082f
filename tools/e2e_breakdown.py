"""Where the end-to-end step time goes (config 2, B=256): the fused step timed by wall clock over 60
steps with (a) device-resident indices, (b) host indices (pinned H2D copy per step), (c) device indices
+ the per-step loss read-back, (d) both (bench.py's e2e)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

obj = BlstmObjective()
B, T = 256, obj.frames
rng = np.random.default_rng(0)
x = rng.standard_normal((4096, T, obj.input_dim), dtype=np.float32)
y = rng.integers(0, obj.classes, (4096, T), dtype=np.int64)
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
batches = [rng.permutation(4096)[:B] for _ in range(8)]
dev = [torch.from_numpy(b).cuda() for b in batches]


def run(host, readback, n=60):
    pending = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(n):
        if host:
            L.train_step(batches[k % 8], 0.01)
        else:
            L.train_step(dev[k % 8], 0.01, device_idx=True)
        if readback:
            fut = L.loss_async()
            if pending is not None:
                pending()
            pending = fut
    if pending is not None:
        pending()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


for host, rb in ((False, False), (True, False), (False, True), (True, True)):
    run(host, rb, 10)
for rep in range(2):
    for host, rb in ((False, False), (True, False), (False, True), (True, True)):
        print(f"host_idx={host!s:5} readback={rb!s:5}: {run(host, rb):.4f} ms/step")
