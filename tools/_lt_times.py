import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import default_tiers, RewardSpec
from paper_2401_07886_b200.trainer import TrainConfig, run_training
its = 400
cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=its, log_every=its, seed=3)
run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, mode="device")
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["BE200_LIB"])
buf = (ctypes.c_ulonglong * (512 * 16))()
lib.be_debug_lt_times(buf, 512 * 16)
t = np.frombuffer(buf, dtype=np.uint64).reshape(512, 16)[:128, :11].astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "gathered", "forward+TD", "partial written", "ticket", "all arrived", "reduced+applied", "packed", "sums", "sums synced", "adam done"]
for k, n in enumerate(names):
    v = t[:, k]
    v = v[v > 0]
    if len(v) == 0: continue
    r = (v - t0) / 1000.0
    print(f"{n:16s} n={len(r):3d} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f} us")
