"""bench.py's one-process-per-GPU strategies end to end (self-spawned ranks, --same-device so two
ranks share the one B200 of the test box): the fused SSGD group step and the asynchronous ADPSGD
exchange run a few steps and print one well-formed JSON line (a barrier / lock timeout raises)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("strategy", ["ssgd", "adpsgd"])
def test_bench_two_ranks_same_device(strategy):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device", "--strategy", strategy,
           "--steps", "3", "--warmup", "3", "--no-cpu", "--no-library", "--n-seq", "1024", "--layers", "2",
           "--classes", "2048"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["strategy"] == strategy
    assert line["value"] > 0 and line["gpu_launches"] > 0
