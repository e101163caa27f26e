"""Train router policies with the GPU trainer exactly as the reference CLI does.

For each seed: `run_training` on ONE environment with one gradient step per
routed request (the reference's own update-to-data ratio, trainer.py:374-401)
and the shipped training config (config.py:55-78 defaults = TrainConfig()),
200k iterations — the same recipe as the reference-trained fixtures
tests/golden/trained_seed{7,8,9,10}.beqn (tests/golden/make_trained_policy.py).
Writes tests/golden/gpu_trained_seed<s>.beqn; tests/test_policy_parity.py
compares both families statistically (Philox vs PCG64 streams
make the policies themselves differ, so parity is on the evaluation statistics).

usage (GPU box): python tools/train_gpu_policies.py [seeds...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2401_07886_b200 import RewardSpec, default_tiers, save_checkpoint  # noqa: E402
from paper_2401_07886_b200.trainer import TrainConfig, run_training  # noqa: E402


def main():
    seeds = [int(s) for s in sys.argv[1:]] or [7, 8, 9, 10]
    out = {}
    for s in seeds:
        cfg = TrainConfig(seed=s)
        t0 = time.time()
        res = run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=1, updates_per_step=1,
                           pending_capacity=1 << 16)
        torch.cuda.synchronize()
        dt = time.time() - t0
        path = os.path.join(ROOT, "tests", "golden", f"gpu_trained_seed{s}.beqn")
        save_checkpoint(res.net, path)
        out[s] = dict(seconds=dt, iterations=cfg.total_iterations, updates=res.updates,
                      transitions=res.transitions, last_log=res.log[-1].__dict__ if res.log else None)
        print(json.dumps({s: out[s]}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "gpu_policies.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
