"""Policy-quality statistics shared by the policy-parity tests and
tools/train_config3_policies.py: the fraction of trailing-20 windows at >= theta
of peak (evalkit.py:217-241) of a policy rolled out greedily on the eight
reference-generated unpredictable-1 traces (tests/golden/policy_traces.npz,
estimated-rate mode, evalkit.py:154-209), and the config-3 training recipe."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THETAS = (0.90, 0.94, 0.96, 0.98)
SEEDS = (7, 8, 9, 10)

# BASELINE.json configs[2] / SURVEY.md §8d config 3: 4096 lockstep envs, 1,048,576-slot
# device replay, batch 512, 8-256-3 Q-MLP, Adam 1e-4, Huber, target sync 500, epsilon
# 1.0 -> 0.05 over 25 %, warm-up 10k; one update per iteration (= per 4096 env-steps),
# 200k iterations = the reference recipe's number of updates (trainer.py:374-401)
# pending_capacity: decisions a request may stay in flight (exploration overloads tiers
# for long stretches; measured high-water mark in profiles/r2_config3_policies.json)
CONFIG3 = dict(n_envs=4096, batch_size=512, buffer_capacity=1 << 20, iterations=200_000,
               updates_per_step=1, pending_capacity=1 << 16)


def traces():
    return np.load(os.path.join(GOLDEN, "policy_traces.npz"))


def window_fractions_gpu(net, z, device):
    """Mean over the traces of the fraction of windows >= theta, through the
    CUDA rollout (bit-exact to the oracle: tests/test_rollout_gpu.py)."""
    import torch
    from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch,
                                       default_tiers)
    from paper_2401_07886_b200.evalkit import windowed
    tiers, rw = default_tiers(), RewardSpec.default()
    E = z["arrival"].shape[0]
    offs = z["seg_offsets"]
    ss = [z["seg_start"][offs[k]:offs[k + 1]] for k in range(E)]
    sr = [z["seg_rate"][offs[k]:offs[k + 1]] for k in range(E)]
    tb = TraceBatch.from_arrays(z["arrival"], z["task"], ss, sr, device=device)
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    ro = GreedyRollout(tiers, rw, E, tb.ld, enc, estimator_mode="estimated", want_realized=False,
                       device=device)
    o = ro.run(tb, net)
    w = windowed(tb, o.reward).cpu().numpy()
    nw = tb.ld - 20 + 1  # every trace holds ld events
    return np.mean([[float((w[k, :nw] >= th).mean()) for th in THETAS] for k in range(E)], axis=0)


def train_config3(seed, device, iterations=None, timing=None):
    from paper_2401_07886_b200 import RewardSpec, default_tiers
    from paper_2401_07886_b200.trainer import TrainConfig, run_training
    its = int(iterations or CONFIG3["iterations"])
    cfg = TrainConfig(batch_size=CONFIG3["batch_size"], buffer_capacity=CONFIG3["buffer_capacity"],
                      total_iterations=its, log_every=its, seed=seed)
    return run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=CONFIG3["n_envs"],
                        updates_per_step=CONFIG3["updates_per_step"], mode="graph", device=device,
                        pending_capacity=CONFIG3["pending_capacity"], timing=timing)


def welch_ok(ref, dev, slack=0.02):
    """Per theta: |mean difference| <= 2 standard errors (Welch, seed variance) + slack."""
    ref, dev = np.asarray(ref), np.asarray(dev)
    se = np.sqrt(ref.var(axis=0, ddof=1) / len(ref) + dev.var(axis=0, ddof=1) / len(dev))
    diff = np.abs(ref.mean(axis=0) - dev.mean(axis=0))
    return diff <= 2 * se + slack, diff, se
