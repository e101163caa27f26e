"""Training throughput probe (config 3 shape): E envs, 1M replay, batch 512."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import default_tiers, RewardSpec
from paper_2401_07886_b200.trainer import TrainConfig, run_training
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
its = int(sys.argv[2]) if len(sys.argv) > 2 else 500
mode = sys.argv[3] if len(sys.argv) > 3 else "graph"
ups = int(sys.argv[4]) if len(sys.argv) > 4 else 1
router = sys.argv[5] if len(sys.argv) > 5 else "fp64"
cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=its,
                  log_every=its, seed=3)
run_training(default_tiers(), RewardSpec.default(), TrainConfig(batch_size=512, buffer_capacity=1 << 20,
             warmup=10_000, total_iterations=100, log_every=100, seed=3), n_envs=E, mode=mode,
             updates_per_step=ups, router=router)  # warm (module load, allocator)
torch.cuda.synchronize()
t0 = time.time()
tm = {}
res = run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=E, mode=mode, updates_per_step=ups, timing=tm,
                   router=router)
torch.cuda.synchronize()
dt = time.time() - t0
print(f"router={router} mode={mode} E={E} its={its} ups={ups}: loop {tm['loop_ms']:.1f} ms device = {its / tm['loop_ms'] * 1e3:.1f} it/s; "
      f"wall incl. setup {dt:.2f}s  {its/dt:.1f} it/s  {E*its/dt:.3e} env-steps/s  "
      f"updates={res.updates} ({res.updates/dt:.1f}/s) transitions={res.transitions} log={res.log[-1]}")
