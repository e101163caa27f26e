"""Error behaviour of the drop-ins (the reference's ValueError family,
SURVEY.md §8b "Errors"): a policy network whose shape does not match the
environment ("expected input dim", policy.py:111-116), task ids outside the
reward spec (encode / request_reward raise, policy.py:57-58, reward.py:117),
non-integer / out-of-range task arrays, bad step inputs — detected on the host
where possible and by the kernels (BE_EINVAL, raised at the next check) where the
data only exists on the device.  Never a silent wrong answer."""
import numpy as np
import pytest
import torch

import goldens
from helpers import enc_of, reward_of, tiers_of
from paper_2401_07886_b200 import (EnvBatch, GreedyRollout, InvalidParameterError, QNetwork, RewardSpec,
                                   StateEncoding, StepRecords, TraceBatch, default_tiers, route, run_eval)

pytestmark = pytest.mark.gpu


def _golden_setup():
    g = goldens.load("unpredictable-1_mixed1")
    m = g["meta"]
    tb = TraceBatch.from_arrays(g["arrival"], g["task"], list(g["seg_start"]), list(g["seg_rate"]))
    ro = GreedyRollout(tiers_of(m), reward_of(m), 1, tb.ld, enc_of(m), estimator_mode=m["estimator_mode"])
    return g, m, tb, ro


def test_mismatched_network_rejected(cuda):
    g, m, tb, ro = _golden_setup()
    wrong = QNetwork.init_random(1, 3, 256, np.random.default_rng(0))  # 1 task, env has 4
    with pytest.raises(ValueError, match="expected input dim"):
        ro.run(tb, wrong)
    wrong_tiers = QNetwork.init_random(4, 2, 256, np.random.default_rng(0))
    with pytest.raises(ValueError):
        ro.run(tb, wrong_tiers)
    # the step API and the batched router check the same
    env = EnvBatch(tiers_of(m), reward_of(m), 2, enc_of(m), estimator_mode="true-rate", ring_capacity=64)
    rec = StepRecords(2, 8, cuda)
    arr = torch.ones(2, dtype=torch.float64, device=cuda)
    tsk = torch.zeros(2, dtype=torch.uint8, device=cuda)
    with pytest.raises(ValueError, match="expected input dim"):
        env.step(arr, tsk, rec, true_rate=torch.ones(2, dtype=torch.float64, device=cuda), policy=wrong)
    with pytest.raises(ValueError):
        route(wrong, torch.zeros((3, 8), dtype=torch.float64, device=cuda))


def test_task_ids_out_of_range(cuda):
    g, m, tb, ro = _golden_setup()
    with pytest.raises(InvalidParameterError):
        TraceBatch.from_arrays(g["arrival"], np.full(len(g["arrival"]), 300), [0], [1.0])
    with pytest.raises(InvalidParameterError):
        TraceBatch.from_arrays(g["arrival"], -np.ones(len(g["arrival"]), np.int64), [0], [1.0])
    with pytest.raises(InvalidParameterError):
        TraceBatch.from_arrays(g["arrival"], np.full(len(g["arrival"]), 0.5), [0], [1.0])
    # a batch whose ids exceed the reward spec: refused before launch ...
    bad = TraceBatch.from_arrays(g["arrival"], np.full(len(g["arrival"]), 5, np.uint8),
                                 list(g["seg_start"]), list(g["seg_rate"]))
    with pytest.raises(ValueError):
        ro.run(bad, QNetwork.from_any(goldens.net_for(m)))
    # ... and an id planted on the device (no host check can see it) fails the env
    tb.task[0, 1234] = 9
    with pytest.raises(ValueError):
        ro.run(tb, QNetwork.from_any(goldens.net_for(m)))


def test_step_rejects_bad_inputs(cuda):
    tiers, rw = default_tiers(), RewardSpec.default()
    env = EnvBatch(tiers, rw, 4, StateEncoding(4, (128.0, 32.0, 8.0)), estimator_mode="true-rate",
                   ring_capacity=64)
    rec = StepRecords(4, 16, cuda)
    rate = torch.full((4,), 3.0, dtype=torch.float64, device=cuda)
    arr = torch.full((4,), 10.0, dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError):  # wrong dtype
        env.step(arr, torch.zeros(4, dtype=torch.int64, device=cuda), rec, true_rate=rate, static_tier=0)
    with pytest.raises(ValueError):  # too short
        env.step(arr[:2], torch.zeros(2, dtype=torch.uint8, device=cuda), rec, true_rate=rate, static_tier=0)
    with pytest.raises(ValueError):  # true-rate mode needs the rate
        env.step(arr, torch.zeros(4, dtype=torch.uint8, device=cuda), rec, static_tier=0)
    # a task id >= n_tasks is caught by the kernel
    env.step(arr, torch.tensor([0, 1, 9, 2], dtype=torch.uint8, device=cuda), rec, true_rate=rate, static_tier=0)
    with pytest.raises(ValueError):
        env.check()


def test_run_eval_rejects_bad_static_tier(cuda):
    g, m, _, _ = _golden_setup()
    from paper_2401_07886_b200.specs import ArrivalEvent, SegmentMark, WorkloadTrace
    tr = WorkloadTrace([ArrivalEvent(float(t), int(k)) for t, k in zip(g["arrival"][:50], g["task"][:50])],
                       [SegmentMark(0, 3.0)], seed=0)
    with pytest.raises(ValueError):
        run_eval(7, tr, tiers_of(m), reward_of(m), enc_of(m))
