"""Device time of one config-2 gradient (B = 256, paper BLSTM) in the BF16
performance mode and in the FP32-parity mode (3xTF32 tcgen05 GEMMs, fp32
activations), plus the parity mode's GEMM rate.  Prints one JSON object.

  python tools/parity_step.py > profiles/r2_parity_step.json
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_04956_b200.blstm import (BlstmObjective, DeviceDataset, Learner, initial_weights,  # noqa: E402
                                         training_flops_per_frame)

obj = BlstmObjective()
B = 256
rng = np.random.default_rng(0)
x = rng.standard_normal((600, obj.frames, obj.input_dim), dtype=np.float32)
y = rng.integers(0, obj.classes, size=(600, obj.frames))
data = DeviceDataset(x, y)
w0 = initial_weights(obj, 0)
out = {"config": "paper BLSTM, B=256, T=21, 32000 classes (config 2), one gradient (fwd + bwd)"}
for prec in ("bf16", "fp32"):
    L = Learner(obj, data, max_batch=B, theta0=w0, precision=prec)
    idx = torch.arange(B, device="cuda")
    for _ in range(2):
        L.gradient_device(idx, B)
    L.stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if prec == "fp32" else 20
    e0.record(L.stream)
    for _ in range(reps):
        L.gradient_device(idx, B)
    e1.record(L.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = training_flops_per_frame(obj) * B * obj.frames
    out[prec] = {"ms_per_gradient": round(ms, 3), "frames_per_s": round(B * obj.frames / (ms * 1e-3), 1),
                 "algorithmic_tflops": round(flops / (ms * 1e-3) / 1e12, 1), "kernel_launches": L.kernel_count()}
    L.close()
out["fp32_over_bf16_time"] = round(out["fp32"]["ms_per_gradient"] / out["bf16"]["ms_per_gradient"], 2)
print(json.dumps(out, indent=1))
