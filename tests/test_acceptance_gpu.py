"""The reference's acceptance criteria 6-11 (T/test_acceptance.py:272-415) run on the
GPU path and at scale: policies trained by the GPU trainer (config-3 recipe: 4096
lockstep envs, one update per iteration, tests/policy_stats.py), evaluated with the
fused rollout over 256 device-generated traces per scenario (the reference uses 1-3),
statistics from the device reducers (reduce_eval buckets = the stable sweep's rates,
be_reduce_selection, windowed threshold counts).

Criteria 6, 7, 10 and 11 are asserted as the reference states them.  Criteria 8 and 9
(policy-quality directions the reference's own 200k-iteration policies fail, SURVEY.md
§4.3) are measured and written to gpurun_out/acceptance_gpu.json, asserted only for
sanity; DESIGN.md records the outcome.
"""
import json
import os

import numpy as np
import pytest
import torch

import policy_stats as ps
from paper_2401_07886_b200 import (GreedyRollout, ModelTierSpec, RewardSpec, StateEncoding, TaskSpec, TraceBatch,
                                   default_tiers, reduce_eval)
from paper_2401_07886_b200.evalkit import (collapse_rate, riemann_usage, scenario_suite, selection_distribution)
from paper_2401_07886_b200.trainer import TrainConfig, fine_tune, run_training

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E_EVAL = 256
THS = (1.00, 0.99, 0.98, 0.96, 0.94)
REPORT = {}


def _enc():
    return StateEncoding(4, tuple(float(t.max_batch) for t in default_tiers()))


def _train(reward, seed, iterations=200_000, init=None, eps_start=1.0):
    cfg = TrainConfig(batch_size=ps.CONFIG3["batch_size"], buffer_capacity=ps.CONFIG3["buffer_capacity"],
                      total_iterations=iterations, log_every=iterations, seed=seed, epsilon_start=eps_start)
    kw = dict(n_envs=ps.CONFIG3["n_envs"], updates_per_step=1, mode="graph",
              pending_capacity=ps.CONFIG3["pending_capacity"])
    if init is not None:
        return fine_tune(init, reward, cfg, default_tiers(), _enc(), **kw).net
    return run_training(default_tiers(), reward, cfg, _enc(), **kw).net


@pytest.fixture(scope="module")
def trained(cuda):
    return _train(RewardSpec.default(), 7)


def _stable_eval(policy, reward, tiers, cuda, seed=11):
    """Stable sweep (14 rates x 40 s held), reset between segments, true rate."""
    sc = scenario_suite("stable")
    tb = TraceBatch.from_scenario(sc, E_EVAL, 4, seed, device=cuda, buckets=sc.rates)
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in default_tiers()))
    ro = GreedyRollout(tiers, reward, E_EVAL, tb.ld, enc, estimator_mode=sc.estimator_mode,
                       reset_between_segments=True, want_realized=False, device=cuda)
    static = policy if isinstance(policy, int) else -1
    o = ro.run(tb, None if static >= 0 else policy, static)
    red = reduce_eval(tb, o.flags, o.reward, THS, len(sc.rates))
    req = red.bucket_req.sum(0).cpu().numpy()
    mean_r = red.bucket_reward.sum(0).cpu().numpy() / np.maximum(req, 1)
    miss = red.bucket_miss.sum(0).cpu().numpy() / np.maximum(req, 1)
    return sc, tb, o, dict(zip(sc.rates, mean_r)), dict(zip(sc.rates, miss))


def test_criterion6_degenerate_environment_optimality(cuda):
    """The large tier meets the deadline at every trained rate: always-large is optimal."""
    tiers = [ModelTierSpec(0, 2, 4.75, 0.25, 64, tokens_per_request=100, name="small"),
             ModelTierSpec(1, 2, 8.0, 1.0, 16, tokens_per_request=100, name="large")]
    spec = RewardSpec(tasks=(TaskSpec("qa", 40.0),), matrix=((0.5, 1.0),))
    enc = StateEncoding(n_tasks=1, batch_scales=(64.0, 16.0), rate_scale=48.0)
    cfg = TrainConfig(total_iterations=20_000, seed=3, rate_low=0.25, rate_high=2.0, warmup=2_000,
                      buffer_capacity=100_000)
    net = run_training(tiers, spec, cfg, enc, mode="graph").net
    tb = TraceBatch.generate("stable", E_EVAL, 1, 123, rates=(0.25, 0.5, 1.0, 2.0), hold_seconds=40.0,
                             device=cuda)
    ro = GreedyRollout(tiers, spec, E_EVAL, tb.ld, enc, estimator_mode="true-rate",
                       reset_between_segments=True, want_realized=False, device=cuda)
    o = ro.run(tb, net)
    n = tb.n_events if tb.n_events is not None else torch.full((E_EVAL,), tb.ld, device=cuda)
    valid = torch.arange(tb.ld, device=cuda)[None, :] < n[:, None]
    share = float(((o.flags & 0x3F) == 1)[valid].double().mean())
    REPORT["c6_large_share"] = share
    assert share >= 0.95, share


def test_criterion7_policy_vs_baselines_stable(cuda, trained):
    """Mean reward per swept rate within 0.05 of the best static baseline (which runs
    at the baseline batch sizes) and a collapse rate >= 10x the large baseline's."""
    rw = RewardSpec.default()
    sc, _, _, pol_mean, pol_miss = _stable_eval(trained, rw, default_tiers(), cuda)
    base_mean, base_miss = {}, {}
    for k in (0, 1, 2):
        _, _, _, base_mean[k], base_miss[k] = _stable_eval(k, rw, default_tiers(baseline=True), cuda)
    worst = min(pol_mean[r] - max(base_mean[k][r] for k in (0, 1, 2)) for r in sc.rates)
    pc = collapse_rate(pol_miss, sc.rates)
    lc = collapse_rate(base_miss[2], sc.rates)
    REPORT["c7"] = dict(worst_margin=worst, policy_collapse=pc, large_collapse=lc)
    assert worst >= -0.05, worst
    assert lc is not None
    assert (pc is None and sc.rates[-1] >= 10 * lc) or (pc is not None and pc >= 10 * lc), (pc, lc)


def _unpredictable(policy, cuda, tiers, gpu_tiers=None):
    sc = scenario_suite("unpredictable-1")
    tb = TraceBatch.from_scenario(sc, E_EVAL, 4, 21, device=cuda)
    rw = RewardSpec.default()
    ro = GreedyRollout(tiers, rw, E_EVAL, tb.ld, _enc(), estimator_mode=sc.estimator_mode,
                       want_realized=False, device=cuda)
    static = policy if isinstance(policy, int) else -1
    o = ro.run(tb, None if static >= 0 else policy, static)
    red = reduce_eval(tb, o.flags, o.reward, THS, 1)
    return red.win_counts.sum(0).cpu().numpy(), float(o.reward.mean())


def test_criterion8_unpredictable_windows_measured(cuda, trained):
    """Reference direction: policy beats the large baseline on windows >= .99/.98/.96/.94
    and the large baseline has more exact-peak windows.  Measured and reported."""
    cp, _ = _unpredictable(trained, cuda, default_tiers())
    cl, _ = _unpredictable(2, cuda, default_tiers(baseline=True))
    REPORT["c8"] = dict(policy=cp.tolist(), large=cl.tolist(), thresholds=THS,
                        direction=[bool(a > b) for a, b in zip(cp[1:], cl[1:])], peak_large=bool(cl[0] > cp[0]))
    assert cp.sum() > 0 and cl.sum() > 0


def test_criterion10_hardware_utility(cuda, trained):
    """Mean reward per GPU of the policy on 4 GPUs beats the large tier on 8 GPUs
    (hw-utility-8gpu: 8 replicas per tier, baseline batches)."""
    _, mean_pol = _unpredictable(trained, cuda, default_tiers())
    sc8 = scenario_suite("hw-utility-8gpu")
    _, mean_l8 = _unpredictable(2, cuda, sc8.adjust_tiers(default_tiers(baseline=True)))
    u_pol, u_l8 = mean_pol / 4, mean_l8 / 8
    REPORT["c10"] = dict(policy_4gpu=u_pol, large_8gpu=u_l8)
    assert u_pol > u_l8, (u_pol, u_l8)


@pytest.fixture(scope="module")
def soft_policy(cuda, trained):
    return _train(RewardSpec.default().with_kind("soft"), 8, iterations=100_000, init=trained, eps_start=0.25)


def _largest_usage(policy, reward, cuda):
    sc, tb, o, _, _ = _stable_eval(policy, reward, default_tiers(), cuda)
    freq = selection_distribution(tb, sc.rates, 4, 3, flags=o.flags)
    return [riemann_usage(freq, sc.rates, t, 2) for t in range(4)]


def test_criterion9_soft_deadline_usage_measured(cuda, trained, soft_policy):
    """Reference direction: after the soft fine-tune, the task with the widest
    large-vs-medium reward gap (hellaswag) raises its large-tier usage the most."""
    rw = RewardSpec.default()
    hard = _largest_usage(trained, rw, cuda)
    soft = _largest_usage(soft_policy, rw.with_kind("soft"), cuda)
    changes = [(s - h) / max(h, 1e-9) for s, h in zip(soft, hard)]
    REPORT["c9"] = dict(hard=hard, soft=soft, changes=changes,
                        ordering=bool(all(changes[0] > c for c in changes[1:])))
    assert all(np.isfinite(changes))


def test_criterion11_different_deadlines_routing(cuda, trained):
    """Per-task deadlines (different-deadlines scenario): openbookqa's large-tier usage
    rises, copa's falls, versus the uniform-deadline policy."""
    sc = scenario_suite("different-deadlines")
    rw_dd = sc.adjust_rewards(RewardSpec.default())
    dd = _train(rw_dd, 9)
    uni = _largest_usage(trained, RewardSpec.default(), cuda)
    ddu = _largest_usage(dd, rw_dd, cuda)
    names = [t.name for t in RewardSpec.default().tasks]
    ob, co = names.index("openbookqa"), names.index("copa")
    REPORT["c11"] = dict(uniform=uni, different=ddu)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(REPORT, open(os.path.join(ROOT, "gpurun_out", "acceptance_gpu.json"), "w"), indent=1)
    assert ddu[ob] > uni[ob], (uni, ddu)
    assert ddu[co] < uni[co], (uni, ddu)
