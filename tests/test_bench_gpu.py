"""bench.py under the driver's own invocation (--steps 20 --warmup 5): the line
must parse, carry the contract keys, and its in-line oracle parity (strided envs
across the batch, which exercises the large-batch rollout variant) and the
cpu_baseline sample parity must show zero mismatches."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_driver_invocation(cuda):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "5",
           "--envs", "8192", "--requests", "2000", "--cpu-seconds", "2", "--no-training",
           "--parity-envs", "32"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches", "parity"):
        assert k in d, k
    assert d["steps"] == 20 and d["warmup"] == 5 and d["gpu_launches"] == 60
    assert d["parity"]["mismatches"] == 0 and d["parity"]["envs"] >= 32
    assert d["cpu_baseline"]["parity"]["mismatches"] == 0 and d["cpu_baseline"]["parity"]["envs"] > 0
    assert d["e2e"]["stats_identical_to_resident_run"]
    assert sum(d["results"]["requests"]) == 8192 * 2000
    assert 0 < d["roofline"]["frac"] < 1
