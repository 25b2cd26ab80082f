"""Per-tile timeline of one GEMM launch of the paper-size training step
(B=256): for every CTA pair, when the MMA issuer started / finished each
tile, how long it stalled on TMA data (full barriers), when the epilogue of
the tile started / finished, and how long the producer waited for free
stages.  Tells a mainloop-bound launch (MMA busy, no full stalls) from a
TMA-latency-bound one (full stalls) and an epilogue-bound one (the MMA
waiting for a drained accumulator between tiles).

  python tools/gemm_trace.py [launch index ...]
launch indices in step order: 0-5 forward layer inputs, 6 bottleneck,
7 CE statistics, 8 dW_o, 9 (dW_b, dY), 10-15 backward layers 5..0.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective, DeviceDataset, Learner, initial_weights  # noqa: E402

TILES, FIELDS = 32, 11
B = 256
lib = _lib.load()
obj = BlstmObjective()
rng = np.random.default_rng(0)
x = rng.standard_normal((2048, 21, 260), dtype=np.float32)
y = rng.integers(0, 32000, size=(2048, 21))
L = Learner(obj, DeviceDataset(x, y), max_batch=B, theta0=initial_weights(obj, 0))
idx = torch.arange(B, device="cuda")
for _ in range(3):
    L.gradient_device(idx, B)
torch.cuda.synchronize()
L.set_profile(True)  # eager launches (no graph), so the traced launch is a live one
buf = torch.zeros(160 * TILES * FIELDS, dtype=torch.int64, device="cuda")
launches = [int(a) for a in sys.argv[1:]] or [1, 7, 8, 10]
for li in launches:
    buf.zero_()
    L.gradient_device(idx, B)  # warm the profiled path
    torch.cuda.synchronize()
    _lib.check(lib.ds_debug_gemm_trace(buf.data_ptr(), li))
    L.gradient_device(idx, B)
    torch.cuda.synchronize()
    _lib.check(lib.ds_debug_gemm_trace(None, 0))
    L.profile_read()
    t = buf.cpu().numpy().reshape(160, TILES, FIELDS).astype(np.float64)
    ctas = int((t[:, 0, 7] > 0).sum())
    t = t[:ctas]
    t0 = t[:, 0, 7].min()
    lead = t[0::2]
    ntile = (lead[:, :, 0] > 0).sum(axis=1)
    print(f"== launch {li}: {ctas} CTAs, tiles per pair min {ntile.min()} max {ntile.max()}")
    start = np.where(lead[:, :, 0] > 0, lead[:, :, 0] - t0, np.nan) / 1e3
    end = np.where(lead[:, :, 2] > 0, lead[:, :, 2] - t0, np.nan) / 1e3
    fst = np.where(lead[:, :, 0] > 0, lead[:, :, 1], np.nan) / 1.9e3  # cycles -> us at ~1.9 GHz
    es = np.where(lead[:, :, 3] > 0, lead[:, :, 3] - t0, np.nan) / 1e3
    ee = np.where(lead[:, :, 4] > 0, lead[:, :, 4] - t0, np.nan) / 1e3
    el = np.where(lead[:, :, 5] > 0, lead[:, :, 5] - t0, np.nan) / 1e3
    pst = np.where(lead[:, :, 0] > 0, t[0::2, :, 6], np.nan) / 1.9e3
    first = (t[:, 0, 7] - t0) / 1e3
    span = np.nanmax(el)
    print(f"  CTA start spread {first.max():.2f} us; last epilogue done {span:.2f} us")
    print(f"  first MMA start: median {np.nanmedian(start[:, 0]):.2f} max {np.nanmax(start[:, 0]):.2f} us")
    print(f"  mainloop per tile (MMA start->end): median {np.nanmedian(end - start):.2f} us, "
          f"TMA-wait stall per tile median {np.nanmedian(fst):.2f} us")
    gap = start[:, 1:] - end[:, :-1]
    print(f"  MMA idle between tiles (accumulator not drained): median {np.nanmedian(gap):.2f} "
          f"max {np.nanmax(gap):.2f} us")
    print(f"  epilogue per tile (warp 0 start->end): median {np.nanmedian(ee - es):.2f} us; "
          f"start->last warp {np.nanmedian(el - es):.2f} us; MMA end->epi start {np.nanmedian(es - end):.2f} us")
    print(f"  producer empty-wait per tile median {np.nanmedian(pst):.2f} us")
    for p in range(min(3, len(lead))):
        row = " | ".join(f"{start[p, i]:6.2f}-{end[p, i]:6.2f} e{es[p, i]:6.2f}-{el[p, i]:6.2f} st{fst[p, i]:4.2f}"
                         for i in range(ntile[p]))
        print(f"  pair {p}: {row}")
