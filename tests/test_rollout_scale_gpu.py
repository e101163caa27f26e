"""Parity of the fused rollout at the batch sizes the bench and BASELINE configs
2/4/5 run (evalkit.py:154-209 per env, simcore.py:113-149 per replica): the
large-batch variants (true-rate throughput variant with the skip table read
through L1; estimated-rate 2-CTA variant), checked on strided env samples
against the C oracle bit for bit.  The launch plan is read back from the handle
(be_env_rollout_plan) so each test proves which variant it exercised."""
import os

import numpy as np
import pytest
import torch

import goldens
from helpers import assert_rows_match_oracle, oracle_rows
from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch,
                                   default_tiers, load_checkpoint, specs)

pytestmark = pytest.mark.gpu
POLICY = os.path.join(goldens.GOLDEN, "trained_seed7.beqn")


def _strided(E, k):
    return sorted(set(np.linspace(0, E - 1, k).round().astype(int).tolist()))


def _run(tb, rw, est, reset=False, want_realized=True):
    tiers = default_tiers()
    enc = StateEncoding(rw.n_tasks, tuple(float(t.max_batch) for t in tiers))
    net = load_checkpoint(POLICY)
    ro = GreedyRollout(tiers, rw, tb.n_envs, tb.ld, enc, estimator_mode=est,
                       reset_between_segments=reset, want_realized=want_realized)
    o = ro.run(tb, net)
    return ro, o, dict(tiers=tiers, reward=rw, net=net, batch_scales=enc.batch_scales,
                       rate_scale=enc.rate_scale, estimator_mode=est, reset=reset)


def _check(tb, o, rw, rows, kw):
    refs = oracle_rows(tb, rows, **kw)
    dl = [t.deadline_ms_per_token for t in rw.tasks]
    task = tb.task.cpu().numpy()
    assert_rows_match_oracle(o, refs, dl, lambda r: task[r])


def test_headline_variant_bench_workload(cuda):
    """Config 4's kernel: 10,000 true-rate envs (more than two waves of the latency
    variant) at load 1x-10x, the reference-trained policy -> rollout_kernel<3, 16,
    TR=1, OCC=1>, skip table through L1, certified screen; 40 strided envs (first, last
    and between, i.e. envs pulled early and late from the dynamic env counter) vs the
    oracle."""
    E, N = 10000, 2000
    rates = [3.0 * (1 + (g % 10)) for g in range(E)]
    tb = TraceBatch.generate_stable(rates, N, 4, 2401, device=cuda, buckets=[g % 10 for g in range(E)])
    rw = RewardSpec.default()
    ro, o, kw = _run(tb, rw, "true-rate")
    plan = ro.env.rollout_plan()
    assert plan["throughput_variant"] == 1 and plan["true_rate"] == 1, plan
    assert plan["lanes_per_env"] == 16 and plan["skip_smem"] == 0 and plan["screen"] == 1, plan
    assert plan["ctas_per_sm"] >= 3, plan
    _check(tb, o, rw, _strided(E, 40), kw)


def test_headline_variant_offset_envs(cuda):
    """A GPU's shard of the sharded config 4 (global ids 57,344..65,535 on rank 7
    of 8): traces keyed by global id; at 8,192 envs two waves of the latency variant
    (2 CTAs/SM, skip table in shared memory) are the shorter makespan; oracle parity."""
    E, N, off = 8192, 1500, 57344
    gids = range(off, off + E)
    tb = TraceBatch.generate_stable([3.0 * (1 + (g % 10)) for g in gids], N, 4, 2401, device=cuda,
                                    env_offset=off)
    rw = RewardSpec.default()
    ro, o, kw = _run(tb, rw, "true-rate", want_realized=False)
    plan = ro.env.rollout_plan()
    assert plan["throughput_variant"] == 0 and plan["true_rate"] == 1, plan
    _check(tb, o, rw, _strided(E, 24), kw)


def _mixed_reward():
    base = RewardSpec.default()
    tasks = tuple(specs.TaskSpec(t.name, t.deadline_ms_per_token, "soft" if k < 2 else "hard")
                  for k, t in enumerate(base.tasks))
    return RewardSpec(tasks=tasks, matrix=base.matrix)


def test_config2_unpredictable_mixed_deadlines(cuda):
    """Config 2: 4,096 envs, 4 tasks with soft (0, 1) and hard (2, 3) deadlines,
    device-generated unpredictable-1 traces (bursty, time-varying), estimated rate."""
    E = 4096
    tb = TraceBatch.generate("unpredictable-time", E, 4, 77, n_requests=2500, device=cuda)
    rw = _mixed_reward()
    ro, o, kw = _run(tb, rw, "estimated")
    plan = ro.env.rollout_plan()
    assert plan["true_rate"] == 0 and plan["screen"] == 1, plan
    _check(tb, o, rw, _strided(E, 32), kw)


@pytest.mark.parametrize("scenario", ["unpredictable-2", "single-task-2", "hellaswag-copa-soft"])
def test_config5_shift_scenarios_at_scale(cuda, scenario):
    """Config 5 (arrival- and task-distribution shift) at 65,536 envs: the scenario
    suite's traces generated on the device (make_trace, evalkit.py:141-151), the
    scenario's estimator / reset / reward kind, strided envs vs the oracle."""
    from paper_2401_07886_b200.evalkit import scenario_suite
    sc = scenario_suite(scenario)
    E = 65536
    kw_gen = {}
    if sc.workload == "stable":
        kw_gen = dict(rates=sc.rates[:10], hold_seconds=20.0)  # ~1,050 requests: the oracle stays quick
    else:
        kw_gen = dict(n_requests=1500)
    tb = TraceBatch.generate(sc.workload, E, 4, 5, task_ids=sc.task_ids, device=cuda, **kw_gen)
    rw = sc.adjust_rewards(RewardSpec.default())
    ro, o, kw = _run(tb, rw, sc.estimator_mode, reset=sc.reset_between_segments, want_realized=False)
    plan = ro.env.rollout_plan()
    assert plan["true_rate"] == (1 if sc.estimator_mode == "true-rate" else 0)
    if sc.estimator_mode == "true-rate":
        assert plan["throughput_variant"] == 1
    _check(tb, o, rw, _strided(E, 24), kw)
