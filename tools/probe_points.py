"""Read the BE_PROBE points of a probe build (development aid).

usage: BE200_LIB=.../lib_P.so python tools/probe_points.py [iterations] [mode]
Runs the config-3 training loop, then prints per probe point the min / median / max
over CTAs of the time since the earliest CTA's point 0 (the last iteration's launch)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_07886_b200 import RewardSpec, default_tiers  # noqa: E402
from paper_2401_07886_b200.trainer import TrainConfig, run_training  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
mode = sys.argv[2] if len(sys.argv) > 2 else "device"
cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=its, log_every=its,
                  seed=3)
run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, mode=mode)
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["BE200_LIB"])
buf = (ctypes.c_ulonglong * (1024 * 16))()
lib.be_debug_probe(buf, 1024 * 16)
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
rows = t[t[:, 0] > 0]
t0 = rows[:, 0].min()
for k in range(16):
    v = rows[:, k]
    v = v[v >= t0]
    if len(v) == 0:
        continue
    r = (v - t0) / 1000.0
    print(f"point {k:2d}  n={len(r):4d}  min {r.min():8.2f}  med {np.median(r):8.2f}  max {r.max():8.2f} us")
