"""Per-load rollout cost (config-4 workload): for each load multiplier L the fused
rollout over E envs all at load L x 3 req/s (10k requests each), and the whole-batch
throughput at the per-GPU env counts of config 4 split over N GPUs (65,536 / N).
Informs the env scheduling order of the persistent rollout (longest first).
usage: python tools/probe_env_cost.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch, default_tiers,  # noqa: E402
                                   load_checkpoint)

dev = torch.device("cuda", 0)
net = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn"))
enc = StateEncoding(4, (128.0, 32.0, 8.0))


def timed(E, rates, N=10000, reps=3):
    tb = TraceBatch.generate_stable(rates, N, 4, 2401, device=dev)
    ro = GreedyRollout(default_tiers(), RewardSpec.default(), E, N, enc, estimator_mode="true-rate",
                       want_realized=False, device=dev)
    ro.run(tb, net)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        ro.launch(tb, net)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = {}
E = 7104  # one env per persistent group of the throughput variant
for L in range(1, 11):
    ms = timed(E, [3.0 * L] * E)
    out[f"load{L}_ms_per_env_wave"] = ms
    print(json.dumps({"load": L, "ms": ms}), flush=True)
for n in (1, 2, 4, 8):
    Eg = 65536 // n
    ms = timed(Eg, [3.0 * (1 + g % 10) for g in range(Eg)])
    out[f"split{n}"] = dict(envs=Eg, ms=ms, steps_per_s=Eg * 10000 / ms * 1e3)
    print(json.dumps({"gpus": n, "envs": Eg, "ms": ms, "per_gpu_steps_per_s": Eg * 10000 / ms * 1e3}), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "env_cost.json"), "w"), indent=1)
