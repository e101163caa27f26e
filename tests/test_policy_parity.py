"""Statistical parity of GPU-trained policies with reference-trained ones
(BASELINE north star: "a trained policy's peak-performance fractions must match
within a stated statistical tolerance").

Policies (all 200k iterations, shipped config, one env, one update per routed
request):
  reference: tests/golden/trained_seed{7,8,9,10}.beqn — the unmodified
             reference trainer (tests/golden/make_trained_policy.py);
  GPU:       tests/golden/gpu_trained_seed{7,8,9,10}.beqn — run_training on the
             B200 (tools/train_gpu_policies.py).
Both families are evaluated by the oracle (bit-exact restatement of run_eval)
on the same eight reference-generated unpredictable-1 traces
(tests/golden/policy_traces.npz).  Statistic per policy: the fraction of
trailing-20 windows >= theta of peak for theta in {0.90, 0.94, 0.96, 0.98},
averaged over the traces.  Tolerance (stated): for each theta the two family
means differ by at most 2 standard errors of their difference (Welch, seed
variance) plus 0.02 absolute.  PCG64 vs Philox streams make the individual
policies differ, so this is the strongest claim available.
"""
import glob
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2401_07886_b200.specs import DEFAULT_TIERS, RewardSpec, load_checkpoint

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THETAS = (0.90, 0.94, 0.96, 0.98)
SEEDS = (7, 8, 9, 10)


def fractions(path, z):
    net = load_checkpoint(path)
    rw = RewardSpec.default()
    out = []
    for k in range(z["arrival"].shape[0]):
        o0, o1 = z["seg_offsets"][k], z["seg_offsets"][k + 1]
        r = oracle.run_eval_oracle(tiers=DEFAULT_TIERS, reward=rw, arrival=z["arrival"][k],
                                   task=z["task"][k], seg_start=z["seg_start"][o0:o1],
                                   seg_rate=z["seg_rate"][o0:o1], net=net,
                                   estimator_mode="estimated", want_steps=False)
        w = oracle.windowed(r["reward"])
        out.append([oracle.threshold_counts(w, [t])[0] / len(w) for t in THETAS])
    return np.mean(out, axis=0)


def test_gpu_trained_policies_match_reference_statistically():
    gpu = [os.path.join(GOLDEN, f"gpu_trained_seed{s}.beqn") for s in SEEDS]
    if not all(os.path.exists(p) for p in gpu):
        pytest.skip("GPU-trained policies not generated yet (tools/train_gpu_policies.py)")
    z = np.load(os.path.join(GOLDEN, "policy_traces.npz"))
    ref = np.array([fractions(os.path.join(GOLDEN, f"trained_seed{s}.beqn"), z) for s in SEEDS])
    dev = np.array([fractions(p, z) for p in gpu])
    se = np.sqrt(ref.var(axis=0, ddof=1) / len(ref) + dev.var(axis=0, ddof=1) / len(dev))
    diff = np.abs(ref.mean(axis=0) - dev.mean(axis=0))
    for k, th in enumerate(THETAS):
        assert diff[k] <= 2 * se[k] + 0.02, (
            f"theta {th}: reference {ref[:, k].round(4)} vs GPU {dev[:, k].round(4)}")
