"""Regenerate the committed golden vectors (run in the build container where
/root/reference is importable).  Every vector is produced by the reference
package itself or by the oracle cross-checked here against torch float64.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import blstm_ref as O  # noqa: E402


def blstm_tiny():
    spec = O.TINY
    x, y, _, _ = O.make_dataset(spec, 8, 7)
    w = O.initial_weights(spec, 7)
    loss, grad = O.loss_and_grad(spec, w, x[:4], y[:4])
    np.savez_compressed(os.path.join(HERE, "blstm_tiny.npz"), spec=np.array(
        [spec.layers, spec.input_dim, spec.hidden, spec.bottleneck, spec.classes, spec.frames]),
        w=w, x=x[:4], y=y[:4], loss=loss, grad=grad)


if __name__ == "__main__":
    blstm_tiny()
    if "--schedule" in sys.argv or True:
        from make_schedule_golden import main as sched  # noqa: E402

        sched()
