"""run_training / fine_tune as drop-ins: the reference's own TestRunTraining and
TestFineTune cases (T/test_trainer.py:186-264) through the GPU trainer, on the
reference's toy environment (2 tiers, 1 task, hidden 8/16 — widths the fused
kernels handle without the fp32 screen), plus the data-parallel-free
updates_per_step = 0 path."""
import numpy as np
import pytest

from paper_2401_07886_b200 import ModelTierSpec, QNetwork, RewardSpec, TaskSpec
from paper_2401_07886_b200.trainer import TrainConfig, fine_tune, run_training

pytestmark = pytest.mark.gpu


def toy_env():  # T/test_trainer.py:23-27
    tiers = [ModelTierSpec(0, 1, 4.75, 0.25, 16, tokens_per_request=10),
             ModelTierSpec(1, 1, 8.0, 1.2, 8, tokens_per_request=10)]
    spec = RewardSpec(tasks=(TaskSpec("qa", 40.0),), matrix=((0.5, 1.0),))
    return tiers, spec


def request_reward(task, tier, realized, spec):
    """reward.py:94-126 restated for the hard-deadline toy spec."""
    t = spec.tasks[task]
    w = 1.0 if realized <= t.deadline_ms_per_token else 0.0
    return w * spec.matrix[task][tier]


def test_zero_iterations_returns_init_unchanged(cuda):
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=0, batch_size=4, warmup=4, buffer_capacity=16, seed=3, hidden=8)
    init = QNetwork.init_random(1, 2, 8, np.random.default_rng(99))
    res = run_training(tiers, spec, cfg, init_net=init)
    for a, b in zip(res.net.params(), init.params()):
        assert np.array_equal(a, b)


def test_deterministic_under_seed(cuda):
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=1500, batch_size=32, warmup=64, buffer_capacity=4096, seed=11,
                      hidden=16, log_every=250, rate_low=0.5, rate_high=8.0)
    r1 = run_training(tiers, spec, cfg)
    r2 = run_training(tiers, spec, cfg)
    assert len(r1.log) == 6 and [row.loss for row in r1.log] == [row.loss for row in r2.log]
    assert np.isfinite(r1.log[-1].loss)
    for a, b in zip(r1.net.params(), r2.net.params()):
        assert np.array_equal(a, b)


def test_rewards_match_completion_records(cuda):
    """completion_log rows (id, task, tier, realized, reward) are consistent with
    request_reward, and every completed request of the run is logged once."""
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=2000, batch_size=32, warmup=64, buffer_capacity=4096, seed=5,
                      hidden=16, rate_low=0.5, rate_high=8.0)
    audit = []
    res = run_training(tiers, spec, cfg, completion_log=audit)
    assert len(audit) > 1000
    ids = [row[0] for row in audit]
    assert len(set(ids)) == len(ids) and max(ids) < 2000
    assert res.transitions <= len(audit)
    rng = np.random.default_rng(0)
    for idx in rng.integers(0, len(audit), size=1000):
        _, task, tier, realized, placed = audit[idx]
        assert task == 0 and tier in (0, 1)
        assert placed == request_reward(task, tier, realized, spec)
        assert 0.0 <= placed <= 1.0
    # the audit trail does not change the training (host-driven vs graph mode)
    ref = run_training(tiers, spec, cfg, mode="graph")
    for a, b in zip(res.net.params(), ref.net.params()):
        assert np.array_equal(a, b)


def test_dimension_mismatch_rejected(cuda):
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=10, batch_size=4, warmup=4, buffer_capacity=16, seed=0)
    wrong = QNetwork.init_random(3, 3, 8, np.random.default_rng(0))
    with pytest.raises(ValueError):
        run_training(tiers, spec, cfg, init_net=wrong)


def test_fine_tune_unchanged_rewards_no_collapse(cuda):
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=4000, batch_size=32, warmup=64, buffer_capacity=4096, seed=2,
                      hidden=16, rate_low=0.5, rate_high=4.0)
    first = run_training(tiers, spec, cfg)
    cfg2 = TrainConfig(total_iterations=2000, batch_size=32, warmup=64, buffer_capacity=4096, seed=3,
                       hidden=16, rate_low=0.5, rate_high=4.0, epsilon_start=0.05, epsilon_end=0.05)
    audit = []
    fine_tune(first.net, spec, cfg2, tiers, completion_log=audit)
    before = np.mean([row[4] for row in audit[:500]])
    after = np.mean([row[4] for row in audit[-500:]])
    assert after > before - 0.1


def test_no_updates_advances_once_per_iteration(cuda):
    """updates_per_step = 0: every iteration routes exactly one request per env
    (the iteration counter advances once; nothing is learned)."""
    tiers, spec = toy_env()
    cfg = TrainConfig(total_iterations=300, batch_size=8, warmup=8, buffer_capacity=4096, seed=4, hidden=16,
                      log_every=100)
    init = QNetwork.init_random(1, 2, 16, np.random.default_rng(1))
    out = {}
    for mode in ("host", "device", "graph"):
        out[mode] = run_training(tiers, spec, cfg, init_net=init, n_envs=5, updates_per_step=0, mode=mode)
    for mode, r in out.items():
        assert r.updates == 0, mode
        for a, b in zip(r.net.params(), init.params()):
            assert np.array_equal(a, b), mode
        assert r.transitions == out["host"].transitions > 5 * 200, mode
