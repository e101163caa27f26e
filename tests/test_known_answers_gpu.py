"""The reference's own hand-stepped known answers (pkg/tests/test_simcore.py,
test_reward.py) through the fused GPU rollout (forced actions, one env): the
same cases tests/test_oracle_golden.py checks on the CPU oracle."""
import numpy as np
import pytest
import torch

from helpers import reward_of, tiers_of
from paper_2401_07886_b200 import GreedyRollout, TraceBatch

pytestmark = pytest.mark.gpu


def _one_tier(alpha, beta, max_batch, tokens, replicas=1):
    return [dict(replicas=replicas, alpha_ms=alpha, beta_ms=beta, max_batch=max_batch,
                 tokens_per_request=tokens)]


HARD40 = dict(tasks=[dict(name="t", deadline=40.0, kind="hard")], matrix=[[1.0]], decay=0.01, cutoff=0.1)


def _run(cuda, tiers, arrivals, reward=HARD40):
    n = len(arrivals)
    meta = dict(tiers=tiers, reward=reward)
    tb = TraceBatch.from_arrays(np.array([arrivals], float), np.zeros((1, n), np.uint8), [[0]], [[1.0]])
    ro = GreedyRollout(tiers_of(meta), reward_of(meta), 1, n, None, estimator_mode="estimated",
                       want_steps=True, ring_capacity=64)
    o = ro.run(tb, forced=torch.zeros((1, n), dtype=torch.uint8, device=cuda))
    return dict(realized=o.realized[0].cpu().numpy(), reward=o.reward[0].cpu().numpy(),
                obs=o.obs[0].cpu().numpy())


def test_single_request_five_ms_per_token(cuda):
    # test_simcore.py:73-79: 100 tokens at alpha 4.75 + beta 0.25 -> 500 ms, 5 ms/token
    assert _run(cuda, _one_tier(4.75, 0.25, 128, 100), [0.0])["realized"][0] == pytest.approx(5.0)


def test_two_simultaneous_share_batch(cuda):
    # test_simcore.py:85-95: two requests share every iteration -> 400 ms, 40 ms/token
    out = _run(cuda, _one_tier(32.0, 4.0, 8, 10), [0.0, 0.0])
    assert list(out["realized"]) == pytest.approx([40.0, 40.0])


def test_queue_wait_counts(cuda):
    # test_simcore.py:109-118: max_batch 1, the second request waits -> 10 and 20 ms/token
    out = _run(cuda, _one_tier(10.0, 0.0, 1, 10), [0.0, 0.0])
    assert list(out["realized"]) == pytest.approx([10.0, 20.0])


def test_completion_at_horizon_counts(cuda):
    # test_simcore.py:103-107, :132-139: an END exactly at the arrival is processed
    # before the arrival observes; observe() == [3] after 99 ms
    assert _run(cuda, _one_tier(4.75, 0.25, 128, 100), [0.0, 500.0])["obs"][1, 0] == 0
    assert _run(cuda, _one_tier(10.0, 0.0, 2, 5), [0.0] * 5 + [99.0])["obs"][5, 0] == 3


def test_min_batch_tie_breaks_low_index(cuda):
    # test_simcore.py:24-36: equal loads -> the lowest replica index takes the request
    out = _run(cuda, _one_tier(4.75, 0.25, 8, 100, replicas=4), [0.0] * 6)
    assert list(out["obs"][:, 0]) == [0, 1, 2, 3, 4, 5]


@pytest.mark.parametrize("ms_per_token,want", [(42.0, 0.98), (44.0, 0.96), (44.01, 0.0), (40.0, 1.0)])
def test_reward_soft_boundaries(cuda, ms_per_token, want):
    # test_reward.py: soft deadline 40 ms/token, decay 0.01, cutoff 10%
    soft = dict(tasks=[dict(name="t", deadline=40.0, kind="soft")], matrix=[[1.0]], decay=0.01, cutoff=0.1)
    out = _run(cuda, _one_tier(ms_per_token, 0.0, 1, 1), [0.0], reward=soft)
    assert out["reward"][0] == pytest.approx(want, abs=1e-12)


@pytest.mark.parametrize("ms_per_token,hit", [(39.9, True), (40.0, True), (40.1, False)])
def test_reward_hard_boundary(cuda, ms_per_token, hit):
    # test_reward.py:24-40: hard deadline 40 ms/token is inclusive
    out = _run(cuda, _one_tier(ms_per_token, 0.0, 1, 1), [0.0])
    assert out["reward"][0] == (1.0 if hit else 0.0)
