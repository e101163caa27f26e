"""Training-loop timing variance: the config-3 loop several times per mode in one process."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import default_tiers, RewardSpec
from paper_2401_07886_b200.trainer import TrainConfig, run_training
its = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
for mode in ("device", "graph", "device", "graph"):
    for rep in range(2):
        cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=its,
                          log_every=its, seed=3 + rep)
        t = {}
        run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, mode=mode, timing=t)
        print(f"{mode} rep{rep}: {its / t['loop_ms'] * 1e3:.0f} it/s ({t['loop_ms']:.1f} ms)", flush=True)
