"""Analysis aid (not product, not a test): how far do BF16 / TF32 / FP32
operand roundings move the paper BLSTM's gradient away from float64?

Runs the float64 oracle (oracle/blstm_ref.py) with every GEMM operand and
the stored activations (gate pre-activations, h, Z, dlogits, dG, dY) rounded
to a given mantissa width, i.e. the rounding points of the device path, and
prints per-block relative L2 errors against the exact float64 gradient.

  python tools/precision_study.py [--batch 16] [--layers 6] [--frames 21]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import blstm_ref as O  # noqa: E402
from oracle.blstm_rounded import loss_and_grad_rounded, rounder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--frames", type=int, default=21)
    ap.add_argument("--classes", type=int, default=32000)
    ap.add_argument("--seed", type=int, default=21)
    args = ap.parse_args()
    spec = O.BlstmSpec(layers=args.layers, frames=args.frames, classes=args.classes)
    x, y, _, _ = O.make_dataset(spec, args.batch, seed=args.seed)
    x = rounder(7)(x)  # device features are bf16 in both modes
    w = O.initial_weights(spec, args.seed)
    l64, g64 = O.loss_and_grad(spec, w, x, y)
    for name, bits in (("fp32", 23), ("tf32", 10), ("bf16", 7)):
        l, g = loss_and_grad_rounded(spec, w, x, y, rounder(bits))
        rel = {}
        for k, (o, shape) in spec.offsets().items() if False else [(k, v) for k, v in spec.offsets().items() if k != "total"]:
            n = int(np.prod(shape))
            a, b = g[o:o + n], g64[o:o + n]
            rel[k] = np.linalg.norm(a - b) / np.linalg.norm(b)
        tot = np.linalg.norm(g - g64) / np.linalg.norm(g64)
        worst = max(rel.items(), key=lambda kv: kv[1])
        print(f"{name}: loss rel {abs(l - l64) / abs(l64):.2e}  grad rel total {tot:.3e}  worst {worst[0]} {worst[1]:.3e}"
              f"  wo {rel['wo']:.3e}  wih0 {rel[('wih', 0)]:.3e}", flush=True)


if __name__ == "__main__":
    main()
