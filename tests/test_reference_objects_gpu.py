"""The drop-in claim with the reference's OWN objects: besteffort's config,
ModelTierSpec / RewardSpec / StateEncoding / QNetwork / WorkloadTrace /
TrainConfig instances (from the unmodified package installed in baseline/_ref)
passed straight into paper_2401_07886_b200.run_eval / run_training
(evalkit.py:154-209, trainer.py:333-406).  run_eval must return the same
records as besteffort.evalkit.run_eval on the same objects.  Skipped when
baseline/_ref is absent."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    if not os.path.isdir(os.path.join(REF, "besteffort")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import besteffort.config
    import besteffort.evalkit
    import besteffort.policy
    import besteffort.trainer
    import besteffort.workload
    return besteffort


def _records(run):
    return [(r.index, r.arrival_ms, r.task_id, r.tier_id, r.reward, r.realized_ms_per_token,
             r.segment_rate) for r in run.records]


@pytest.mark.parametrize("scenario,policy", [("unpredictable-1", "trained"), ("stable", "trained"),
                                             ("hellaswag-copa-soft", "random"), ("unpredictable-2", 1)])
def test_run_eval_with_reference_objects(cuda, be, scenario, policy):
    from paper_2401_07886_b200 import run_eval
    cfg = be.config.parse_config()
    sc = cfg.scenario(scenario)
    tiers, spec, enc = sc.adjust_tiers(cfg.tiers()), sc.adjust_rewards(cfg.reward_spec()), cfg.encoding()
    trace = be.evalkit.make_trace(sc, cfg.n_tasks, 4242)
    if len(trace.events) > 4000:  # keep the reference's Python loop short
        trace = be.workload.WorkloadTrace(trace.events[:4000],
                                          [m for m in trace.segment_marks if m.start_index < 4000],
                                          seed=trace.seed)
    if policy == "trained":
        pol = be.policy.load_checkpoint(os.path.join(GOLDEN, "trained_seed7.beqn"))
    elif policy == "random":
        pol = be.policy.QNetwork.init_random(cfg.n_tasks, cfg.n_tiers, 256, np.random.default_rng(3))
    else:
        pol = policy  # static tier
    kw = dict(estimator_mode=sc.estimator_mode, reset_between_segments=sc.reset_between_segments)
    ref = be.evalkit.run_eval(pol, trace, tiers, spec, enc, **kw)
    got = run_eval(pol, trace, tiers, spec, enc, **kw)
    assert got.policy_id == ref.policy_id and got.gpu_count == ref.gpu_count
    a, b = _records(ref), _records(got)
    assert len(a) == len(b) == len(trace.events)
    for x, y in zip(a, b):
        assert x[:4] == y[:4] and np.float64(x[4]).tobytes() == np.float64(y[4]).tobytes(), (x, y)
        assert np.float64(x[5]).tobytes() == np.float64(y[5]).tobytes() and x[6] == y[6], (x, y)
    # the reference's own reducers accept the drop-in's EvalRun
    th = (1.0, 0.98, 0.96, 0.94, 0.90)
    wa = be.evalkit.windowed(ref.rewards())
    wb = be.evalkit.windowed(got.rewards())
    assert be.evalkit.threshold_counts(wa, th) == be.evalkit.threshold_counts(wb, th)
    assert ref.miss_fractions_by_rate(spec) == got.miss_fractions_by_rate(spec)


def test_run_training_with_reference_objects(cuda, be):
    """The reference TrainConfig / tiers / RewardSpec / init QNetwork go in; the
    trained network comes out as parameters the reference QNetwork accepts."""
    from paper_2401_07886_b200.trainer import run_training
    cfg = be.config.parse_config()
    tc = be.trainer.TrainConfig(total_iterations=600, batch_size=64, warmup=200, buffer_capacity=4096,
                                seed=5, log_every=200)
    init = be.policy.QNetwork.init_random(cfg.n_tasks, cfg.n_tiers, 256, np.random.default_rng(1))
    res = run_training(cfg.tiers(), cfg.reward_spec(), tc, cfg.encoding(), init_net=init)
    assert res.updates > 0 and len(res.log) == 3
    net = be.policy.QNetwork(cfg.n_tasks, cfg.n_tiers, res.net.w1, res.net.b1, res.net.w2, res.net.b2)
    x = np.zeros(cfg.n_tasks + cfg.n_tiers + 1)
    x[0] = 1.0
    assert np.all(np.isfinite(net.forward(x)))
    assert any(not np.array_equal(p, q) for p, q in zip(net.params(), init.params()))
