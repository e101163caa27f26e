"""Small workloads over the kernels added in round 2, for compute-sanitizer
(memcheck / racecheck / synccheck): the fused training iteration (arrivals + step +
replay commit, fp64 and tcgen05 decisions, the commit list overflowing; backward +
Adam in one launch), the split tensor-core form (> 16 replicas), the
completion-range commit, the step split (observe / route_tc / submit), segment
resets, the rollout's device-side task check and the by-value reducer thresholds."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_07886_b200 import (EnvBatch, ModelTierSpec, RewardSpec, StateEncoding, StepRecords,  # noqa: E402
                                   TensorCoreRouter, TraceBatch, GreedyRollout, default_tiers, load_checkpoint,
                                   reduce_eval)
from paper_2401_07886_b200.trainer import TrainConfig, run_training  # noqa: E402

dev = torch.device("cuda", 0)
rw = RewardSpec.default()
cfg = TrainConfig(batch_size=16, buffer_capacity=4096, warmup=16, total_iterations=10, log_every=5, seed=1)
for router in ("fp64", "tc"):
    run_training(default_tiers(), rw, cfg, n_envs=40, mode="device", router=router, pending_capacity=256)
# the fused step + commit with its block list overflowing (list entries + per-env rescan)
os.environ["BE_COMMIT_LIST_CAP"] = "1"
run_training(default_tiers(), rw, cfg, n_envs=40, mode="device", pending_capacity=256)
del os.environ["BE_COMMIT_LIST_CAP"]
wide = [ModelTierSpec(i, 6, t.alpha_ms, t.beta_ms, t.max_batch, t.tokens_per_request) for i, t in
        enumerate(default_tiers())]  # 18 replicas per env: the split tensor-core path
run_training(wide, rw, cfg, StateEncoding(4, (128.0, 32.0, 8.0)), n_envs=24, mode="device", router="tc",
             pending_capacity=256)
net = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn"))
E = 20
env = EnvBatch(default_tiers(), rw, E, StateEncoding(4, (128.0, 32.0, 8.0)), estimator_mode="true-rate",
               ring_capacity=256)
rec = StepRecords(E, 64, dev)
tc = TensorCoreRouter(net, dev)
t = torch.zeros(E, dtype=torch.float64, device=dev)
rate = torch.full((E,), 12.0, dtype=torch.float64, device=dev)
task = torch.arange(E, device=dev).remainder(4).to(torch.uint8)
for i in range(30):
    t += 60.0
    if i == 15:
        env.new_segment(rec, mask=(torch.arange(E, device=dev) % 2).to(torch.uint8))
    o = env.observe(t, task, rec, true_rate=rate)
    _, a = tc(o["x"], want_q=False, check=False)
    env.submit(t, task, a, rec)
env.drain(rec)
env.check()
tb = TraceBatch.generate_stable([6.0] * 64, 300, 4, 3, device=dev, buckets=[0] * 64)
ro = GreedyRollout(default_tiers(), rw, 64, tb.ld, StateEncoding(4, (128.0, 32.0, 8.0)), estimator_mode="true-rate",
                   device=dev)
o = ro.run(tb, net)
red = reduce_eval(tb, o.flags, o.reward, (1.0, 0.98, 0.96), 1)
tb.task[3, 17] = 8
try:
    ro.run(tb, net)
    raise SystemExit("expected the task check to fail")
except ValueError:
    pass
torch.cuda.synchronize()
print("sanitize_r2 ok", red.totals()["requests"])
