"""torch.profiler breakdown of the training loop (kernel vs host time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2401_07886_b200 import default_tiers, RewardSpec
from paper_2401_07886_b200.trainer import TrainConfig, run_training
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=1000, total_iterations=60, log_every=60, seed=3)
run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=E)  # warm
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=E)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15))
