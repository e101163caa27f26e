"""Fixture generator: train the reference router on CPU and save it as BEQN1.

Test infrastructure only. Runs the UNMODIFIED reference trainer
(`pkg/src/besteffort/trainer.py:333` run_training) with the shipped config
(`pkg/src/besteffort/config.py:25-85`), exactly as the acceptance fixture
`trained_policy` does (`pkg/tests/test_acceptance.py:52-58`: seed 7, 200k
iterations).  The resulting checkpoint is committed as
`tests/golden/trained_seed7.beqn` so GPU tests and bench.py use a realistic,
mixed-routing policy without needing the reference at run time.

Usage (in the build container, ~16 min on one core):
    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_trained_policy.py [--tasks 4] [--iters 200000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))

from besteffort.config import parse_config  # noqa: E402
from besteffort.policy import save_checkpoint  # noqa: E402
from besteffort.reward import RewardSpec  # noqa: E402
from besteffort.trainer import run_training  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--iters", type=int, default=200_000)
    ap.add_argument("--tasks", type=int, default=4, help="1 = hellaswag only (config 1)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = parse_config()
    reward = cfg.reward_spec()
    enc = cfg.encoding()
    if a.tasks == 1:
        reward = RewardSpec(tasks=reward.tasks[:1], matrix=reward.matrix[:1])
        from besteffort.policy import StateEncoding
        enc = StateEncoding(n_tasks=1, batch_scales=enc.batch_scales, rate_scale=enc.rate_scale)
    t0 = time.time()
    res = run_training(cfg.tiers(), reward, cfg.train_config(seed=a.seed, total_iterations=a.iters), enc)
    out = a.out or os.path.join(os.path.dirname(__file__),
                                f"trained_seed{a.seed}" + ("_t1" if a.tasks == 1 else "") + ".beqn")
    save_checkpoint(res.net, out)
    print(f"saved {out} after {time.time() - t0:.1f}s; log tail: {res.log[-1] if res.log else None}")


if __name__ == "__main__":
    main()
