"""Golden-vector generator (test infrastructure; run in the build container only).

Imports the UNMODIFIED reference package (read-only, /root/reference/pkg/src)
and records, for a matrix of (scenario, router) runs:

* the trace as SoA arrays (arrival_ms f64, task u8, segment starts/rates);
* the reference `run_eval` records (`pkg/src/besteffort/evalkit.py:154-209`):
  tier, reward, realized ms/token per request;
* per-step router inputs from a harness that replays the run_eval loop
  (`evalkit.py:185-205`) against the reference's own ClusterSim /
  RateEstimator / encode / QNetwork objects: per-tier observed batch
  (`simcore.py:155-157`), rate signal (`workload.py:234-247`), Q-values
  (`policy.py:111-118`) and the fp64 top-2 margin (for tie-aware compare);
* reducer outputs: `windowed` + `threshold_counts` (`evalkit.py:217-241`),
  miss fractions by rate (`evalkit.py:61-68`).

The fixtures are written to tests/golden/*.npz with the numpy version used
(PCG64 streams are not pinned across numpy versions).  The GPU
box never runs this script; it only reads the committed .npz files.

Usage:  python tests/golden/make_golden.py
"""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))

from besteffort import evalkit as ek  # noqa: E402
from besteffort.config import component_seed, parse_config  # noqa: E402
from besteffort.policy import (QNetwork, RouterState, StateEncoding, encode,  # noqa: E402
                               load_checkpoint)
from besteffort.reward import RewardSpec, request_reward  # noqa: E402
from besteffort.simcore import ClusterSim, Request  # noqa: E402
from besteffort.workload import (RateEstimator, WorkloadTrace, ArrivalEvent,  # noqa: E402
                                 SegmentMark, estimate_rate, gen_stable)

HERE = os.path.dirname(os.path.abspath(__file__))


def tiers_json(tiers):
    return [dict(replicas=t.replicas, alpha_ms=t.alpha_ms, beta_ms=t.beta_ms,
                 max_batch=t.max_batch, tokens_per_request=t.tokens_per_request)
            for t in tiers]


def reward_json(spec):
    return dict(tasks=[dict(name=t.name, deadline=t.deadline_ms_per_token, kind=t.kind)
                       for t in spec.tasks],
                matrix=[list(r) for r in spec.matrix], decay=spec.decay_per_ms,
                cutoff=spec.cutoff_fraction)


def mixed_net(s):
    """Random nets that route to all three tiers."""
    net = QNetwork.init_random(4, 3, 256, np.random.default_rng(100 + s))
    net.b2[:] = np.random.default_rng(5 + s).normal(0.0, 0.6, size=3)
    net.w2 *= 3.0
    return net


def harness(policy, trace, tiers, reward_spec, encoding, estimator_mode, reset):
    """Replays evalkit.py:185-205 with the reference objects, recording inputs."""
    n = len(trace.events)
    M = len(tiers)
    obs = np.zeros((n, M), np.int32)
    rate = np.zeros(n)
    q = np.full((n, M), np.nan)
    margin = np.full(n, np.inf)
    static = policy if isinstance(policy, int) else None
    sim = ClusterSim(tiers)
    est = RateEstimator(estimator_mode, 1.0)
    ev_rates = trace.event_rates()
    it = iter(m.start_index for m in trace.segment_marks)
    nb = next(it, None)
    for i, ev in enumerate(trace.events):
        while nb is not None and i >= nb:
            if reset and i == nb and i > 0:
                sim.drain()
                sim = ClusterSim(tiers)
                est.reset()
            nb = next(it, None)
        sim.advance(ev.time_ms)
        est.true_rate = float(ev_rates[i])
        r = estimate_rate(est, ev.time_ms)
        o = sim.observe()
        obs[i] = o
        rate[i] = r
        if static is None:
            qv = policy.forward(encode(RouterState(ev.task_id, tuple(o), r), encoding))
            q[i] = qv
            srt = np.sort(qv)
            margin[i] = srt[-1] - srt[-2]
            tier = int(np.argmax(qv))
        else:
            tier = static
        sim.submit(Request(id=i, task_id=ev.task_id, arrival_ms=ev.time_ms,
                           tokens_target=tiers[tier].tokens_per_request), tier)
    return obs, rate, q, margin


def trace_arrays(trace):
    arr = np.array([e.time_ms for e in trace.events], np.float64)
    task = np.array([e.task_id for e in trace.events], np.uint8)
    ss = np.array([m.start_index for m in trace.segment_marks], np.int64)
    sr = np.array([m.rate for m in trace.segment_marks], np.float64)
    return arr, task, ss, sr


def truncate(trace, n):
    ev = trace.events[:n]
    marks = [m for m in trace.segment_marks if m.start_index < n] or trace.segment_marks[:1]
    return WorkloadTrace(events=ev, segment_marks=marks, seed=trace.seed)


def quantize(trace, q_ms):
    ev = [ArrivalEvent(math.floor(e.time_ms / q_ms) * q_ms, e.task_id) for e in trace.events]
    return WorkloadTrace(events=ev, segment_marks=list(trace.segment_marks), seed=trace.seed)


def run_case(name, policy, policy_name, trace, tiers, reward, enc, scen):
    run = ek.run_eval(policy, trace, tiers, reward, enc, estimator_mode=scen.estimator_mode,
                      reset_between_segments=scen.reset_between_segments)
    tier = np.array([r.tier_id for r in run.records], np.uint8)
    rw = np.array([r.reward for r in run.records])
    rl = np.array([r.realized_ms_per_token for r in run.records])
    obs, rate, q, margin = harness(policy, trace, tiers, reward, enc, scen.estimator_mode,
                                   scen.reset_between_segments)
    w = ek.windowed(rw)
    counts = ek.threshold_counts(w, (1.0, 0.99, 0.98, 0.96, 0.94, 0.90))
    miss = run.miss_fractions_by_rate(reward)
    arr, task, ss, sr = trace_arrays(trace)
    meta = dict(name=name, scenario=scen.name, policy=policy_name, tiers=tiers_json(tiers),
                reward=reward_json(reward),
                enc=dict(batch_scales=list(enc.batch_scales), rate_scale=enc.rate_scale),
                estimator_mode=scen.estimator_mode, reset=scen.reset_between_segments,
                prior_rate=1.0, numpy=np.__version__,
                static_tier=policy if isinstance(policy, int) else -1,
                thresholds=[1.0, 0.99, 0.98, 0.96, 0.94, 0.90],
                counts=[counts[t] for t in (1.0, 0.99, 0.98, 0.96, 0.94, 0.90)],
                n_windows=int(w.size),
                miss_by_rate=[[float(k), float(v)] for k, v in sorted(miss.items())])
    np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"), meta=json.dumps(meta),
                        arrival=arr, task=task, seg_start=ss, seg_rate=sr, tier=tier,
                        reward=rw, realized=rl, obs=obs, rate=rate, q=q, margin=margin,
                        windowed=w)
    mix = np.bincount(tier, minlength=len(tiers))
    print(f"{name:48s} n={len(trace)} mix={mix.tolist()} mean={rw.mean():.4f} "
          f"minmargin={np.min(margin) if policy_name != 'static' else float('nan'):.3g}")


def main():
    cfg = parse_config()
    enc = cfg.encoding()
    nets = {f"mixed{s}": mixed_net(s) for s in range(3)}
    ckpt = os.path.join(HERE, "trained_seed7.beqn")
    if os.path.exists(ckpt):
        nets["trained"] = load_checkpoint(ckpt)
    np.savez_compressed(os.path.join(HERE, "nets.npz"),
                        **{f"{k}_{p}": getattr(v, p) for k, v in nets.items()
                           for p in ("w1", "b1", "w2", "b2")})
    n_short = 2000
    for scen_name in ("stable", "unpredictable-1", "unpredictable-2", "hellaswag-copa-soft",
                      "different-deadlines"):
        scen = cfg.scenario(scen_name)
        if scen.workload == "stable":
            from dataclasses import replace
            scen = replace(scen, hold_seconds=10.0)
        reward = scen.adjust_rewards(cfg.reward_spec())
        trace = truncate(ek.make_trace(scen, cfg.n_tasks, component_seed(0, f"gen:{scen_name}:0")),
                         n_short)
        for pname, net in nets.items():
            if pname == "trained":
                continue
            run_case(f"{scen_name}_{pname}", net, pname, trace,
                     scen.adjust_tiers(cfg.tiers()), reward, enc, scen)
        for k in range(3):
            run_case(f"{scen_name}_static{k}", k, "static", trace,
                     scen.adjust_tiers(cfg.tiers(baseline=True)), reward, enc, scen)
    if "trained" in nets:
        for scen_name in ("unpredictable-1", "unpredictable-2", "stable", "single-task-0",
                          "hw-utility-8gpu", "single-task-3"):
            scen = cfg.scenario(scen_name)
            reward = scen.adjust_rewards(cfg.reward_spec())
            trace = ek.make_trace(scen, cfg.n_tasks, component_seed(0, f"gen:{scen_name}:0"))
            if scen_name not in ("unpredictable-1",):
                trace = truncate(trace, 4000)
            run_case(f"{scen_name}_trained", nets["trained"], "trained", trace,
                     scen.adjust_tiers(cfg.tiers()), reward, enc, scen)
    # config 1 (BASELINE.json configs[0]): one env, 3 tiers x 1 task
    # (hellaswag, hard 40 ms/token), Poisson arrivals, true-rate estimator,
    # greedy DQN over 10k requests; T=1 trained policy + init_random(rng 0)
    ckpt1 = os.path.join(HERE, "trained_seed7_t1.beqn")
    reward1 = RewardSpec(tasks=cfg.reward_spec().tasks[:1], matrix=cfg.reward_spec().matrix[:1])
    enc1 = StateEncoding(n_tasks=1, batch_scales=enc.batch_scales, rate_scale=enc.rate_scale)
    nets1 = {"random_t1": QNetwork.init_random(1, 3, 256, np.random.default_rng(0))}
    if os.path.exists(ckpt1):
        nets1["trained_t1"] = load_checkpoint(ckpt1)
    np.savez_compressed(os.path.join(HERE, "nets_t1.npz"),
                        **{f"{k}_{p}": getattr(v, p) for k, v in nets1.items()
                           for p in ("w1", "b1", "w2", "b2")})
    from dataclasses import replace as _replace
    scen1 = _replace(cfg.scenario("stable"), name="cfg1")
    for lam in (0.25, 4.0, 32.0, 48.0):
        tr = gen_stable([lam], math.ceil(10000 / lam * 1.1), 1,
                        component_seed(0, f"gen:cfg1:{lam}"))
        tr = truncate(tr, 10000)
        for pname, net in nets1.items():
            run_case(f"cfg1_{lam:g}_{pname}", net, pname, tr, cfg.tiers(), reward1, enc1, scen1)
    # tie-forcing: 5 ms quantised arrivals make END == arrival coincidences common
    scen = cfg.scenario("unpredictable-2")
    reward = cfg.reward_spec()
    trace = quantize(truncate(ek.make_trace(scen, cfg.n_tasks,
                                            component_seed(0, "gen:unpredictable-2:0")), 3000), 5.0)
    for pname in ("mixed0", "trained"):
        if pname in nets:
            run_case(f"quantized_{pname}", nets[pname], pname, trace, cfg.tiers(), reward, enc,
                     scen)
    for k in range(3):
        run_case(f"quantized_static{k}", k, "static", trace, cfg.tiers(baseline=True), reward,
                 enc, scen)


if __name__ == "__main__":
    main()
