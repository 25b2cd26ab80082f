"""HBM roofline of the synchronisation kernels at paper size (P = 43.1 M
params), two learners on one device (same-device pointers: the kernels are
the ones the P2P path runs with peer pointers, where NVLink instead of HBM is
the bound).  Prints one JSON object; bytes are algorithmic (each parameter
array element read / written once).

  python tools/sync_bench.py > profiles/r2_sync_kernels.json
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_04956_b200 import _lib  # noqa: E402
from paper_1904_04956_b200.blstm import BlstmObjective  # noqa: E402

P = BlstmObjective().param_dim
lib = _lib.load()
dev = torch.device("cuda", 0)
th = [torch.randn(P, device=dev) * 0.1 for _ in range(2)]
v = [torch.zeros(P, device=dev) for _ in range(2)]
g = [torch.randn(P, device=dev) * 1e-3 for _ in range(2)]
snap = [torch.zeros(P, device=dev, dtype=torch.bfloat16) for _ in range(2)]
flag = torch.zeros(1, device=dev, dtype=torch.int32)
err = torch.zeros(1, device=dev, dtype=torch.int32)
ctl = torch.zeros(16, device=dev, dtype=torch.int32)
dig = torch.zeros(2, device=dev, dtype=torch.int64)
s = torch.cuda.current_stream().cuda_stream


def arr(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = {
    # name: (callable, algorithmic bytes per call)
    "sgd_momentum (v,theta rw + g r)": (
        lambda: _lib.check(lib.ds_sgd_momentum(th[0].data_ptr(), v[0].data_ptr(), g[0].data_ptr(), 0.01, 0.9, P, None,
                                               flag.data_ptr(), s)), 20 * P),
    "adpsgd_mix (both theta rw)": (
        lambda: _lib.check(lib.ds_adpsgd_mix(th[0].data_ptr(), th[1].data_ptr(), P, s)), 16 * P),
    "pair_mix, both halves (theta rw + 2 bf16 snapshots)": (
        lambda: [_lib.check(lib.ds_pair_mix(th[0].data_ptr(), th[1].data_ptr(), snap[0].data_ptr(), snap[1].data_ptr(),
                                             P, h, s)) for h in (0, 1)], 20 * P),
    "shard_step world 2, both ranks (SSGD reduce-scatter + SGD + all-gather)": (
        lambda: [_lib.check(lib.ds_shard_step(2, r, arr(g), arr(th), arr(snap), v[r].data_ptr(), P, 2, 0.01, 0.9, 0,
                                               0.0, s)) for r in (0, 1)], 32 * P),
    "update_mix (N1: sgd_step + pair average in one pass; theta,v rw + g r + snapshot w + peer rw)": (
        lambda: _lib.check(lib.ds_update_mix(th[0].data_ptr(), v[0].data_ptr(), g[0].data_ptr(), th[1].data_ptr(),
                                             snap[0].data_ptr(), 0.01, 0.9, P, flag.data_ptr(), s)), 30 * P),
    "sgd_momentum + adpsgd_mix unfused (the N1 baseline)": (
        lambda: (_lib.check(lib.ds_sgd_momentum(th[0].data_ptr(), v[0].data_ptr(), g[0].data_ptr(), 0.01, 0.9, P,
                                                None, flag.data_ptr(), s)),
                 _lib.check(lib.ds_adpsgd_mix(th[0].data_ptr(), th[1].data_ptr(), P, s))), 30 * P),
    "digest (debug WeightMessage checksum, theta read)": (
        lambda: _lib.check(lib.ds_digest(th[0].data_ptr(), 4 * P, dig.data_ptr(), s)), 4 * P),
    "peer lock + unlock (empty critical section)": (
        lambda: (_lib.check(lib.ds_peer_lock(ctl.data_ptr(), 1, err.data_ptr(), 5.0, s)),
                 _lib.check(lib.ds_peer_unlock(ctl.data_ptr(), s))), 0),
    "group_reduce world 2, both owners (single-process SSGD)": (
        lambda: [_lib.check(lib.ds_group_reduce(2, r, arr(g), arr(th), arr(v), None, P, 2, 0.01, 0.9, 0, 0.0, s))
                 for r in (0, 1)], 36 * P),
}
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = None
out = {"param_dim": P, "hbm_peak_gbs": peak, "kernels": {}}
for name, (fn, nbytes) in cases.items():
    ms = timed(fn)
    gbs = nbytes / (ms * 1e-3) / 1e9
    out["kernels"][name] = {"ms": round(ms, 4), "bytes": nbytes, "GB/s": round(gbs, 1),
                            "frac_of_hbm": round(gbs / peak, 3) if peak and nbytes else None}
print(json.dumps(out, indent=1))
