import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import default_tiers, RewardSpec, _lib
from paper_2401_07886_b200.trainer import TrainConfig, run_training
its = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=its, log_every=its, seed=3)
mode = sys.argv[2] if len(sys.argv) > 2 else "device"
tm = {}
run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, mode=mode, timing=tm)
print(mode, its / tm["loop_ms"] * 1e3, "it/s")
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["BE200_LIB"])
buf = (ctypes.c_ulonglong * (1024 * 8))()
lib.be_debug_stepc_times(buf, 1024 * 8)
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8)[:256].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["start", "publish", "step_end", "lookback_end", "after_bar", "writes_end", "round_end"]
for k, n in enumerate(names):
    v = rel[:, k]
    print(f"{n:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
print("per-CTA durations (median / max):")
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6)]:
    d = rel[:, b] - rel[:, a]
    print(f"  {names[a]:>12s} -> {names[b]:12s} med {np.median(d):7.2f} max {d.max():7.2f}  argmax CTA {int(d.argmax())}")
lg = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8)[:256, 7]
print("max range L per CTA (top 8):", np.sort(lg >> np.uint64(32))[-8:], " max gtot:", np.sort(lg & np.uint64(0xffffffff))[-8:])
print("late starters:", np.argsort(-rel[:, 0])[:8], np.sort(rel[:, 0])[-8:])
print("late publishers:", np.argsort(-rel[:, 1])[:8], np.sort(rel[:, 1])[-8:])
