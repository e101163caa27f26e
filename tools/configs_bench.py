"""Every BASELINE.json configuration on one B200 (results -> gpurun_out/configs.json).

  config 1  single env, T = 1 (hellaswag), 9 arrival rates 0.25..48 req/s, stable
            Poisson truncated to 10k requests, true-rate estimator, trained T = 1
            policy and a random-init one: the latency of ONE env through run_eval
            (the drop-in), and all 18 (rate, policy) envs batched in one launch
  config 2  4096 envs, 3 models x 4 tasks with hard/soft deadlines
            (hellaswag/piqa hard, copa/openbookqa soft, 40 ms/token),
            time-varying bursty unpredictable-1 traces, estimated rate, greedy
  config 3  training: 4096 envs, 1M replay, batch 512, Adam (updates/s)
  config 4  the bench.py workload (65,536 envs, load 1x-10x)
  config 5  robustness on 65,536 envs: arrival shift (unpredictable-2, and
            unpredictable-1) and task shift (single-task-0..3, and the
            {hellaswag, copa} soft subset), same trained policy
Traces are generated on the device (Philox); env-steps/s are device time of the
fused rollout; statistics from the on-device reducer (windows >= theta of peak,
availability = 1 - deadline-miss fraction).
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_07886_b200 import (GreedyRollout, QNetwork, RewardSpec, StateEncoding, TaskSpec,  # noqa: E402
                                   TraceBatch, default_tiers, load_checkpoint, reduce_eval, run_eval)
from paper_2401_07886_b200.evalkit import scenario_suite  # noqa: E402
from paper_2401_07886_b200.specs import DEFAULT_MATRIX  # noqa: E402
from paper_2401_07886_b200.trainer import TrainConfig, run_training  # noqa: E402

TH = (1.00, 0.98, 0.96, 0.94, 0.90)
POL = os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn")
POL_T1 = os.path.join(ROOT, "tests", "golden", "trained_seed7_t1.beqn")


def timed_rollout(ro, tb, net, reps=3):
    ro.run(tb, net)  # warm + settle the ring capacity
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o = ro.launch(tb, net)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ro.env.check()
    return o, min(ms)


def stats(red):
    t = red.totals()
    req, miss = np.array(t["requests"]), np.array(t["misses"])
    return dict(window_fraction=dict(zip([str(x) for x in TH], t["window_fraction"])),
                availability=float(1 - miss.sum() / max(req.sum(), 1)),
                availability_by_bucket=t["availability"], requests=int(req.sum()))


def config1():
    tiers = default_tiers()
    rw = RewardSpec(tasks=(TaskSpec("hellaswag", 40.0, "hard"),), matrix=(DEFAULT_MATRIX[0],))
    enc = StateEncoding(1, tuple(float(t.max_batch) for t in tiers))
    rates = [0.25, 1, 2, 4, 8, 16, 24, 32, 48]
    trained = load_checkpoint(POL_T1)
    rand = QNetwork.init_random(1, 3, 256, np.random.default_rng(0))
    tb = TraceBatch.generate("stable", len(rates), 1, seed=101, rates=[[r] for r in rates],
                             hold_seconds=math.ceil(10000 / min(rates) * 1.1), ld=10000, truncate=True,
                             buckets=rates)
    out = {}
    # one env through the drop-in run_eval (records back on the host)
    tr = tb.to_workload_trace(3)
    run_eval(trained, tr, tiers, rw, enc, estimator_mode="true-rate")
    ts = []
    for _ in range(5):  # median of 5 (wall clock: env setup, kernel, 10k host records)
        t0 = time.perf_counter()
        run_eval(trained, tr, tiers, rw, enc, estimator_mode="true-rate")
        ts.append(time.perf_counter() - t0)
    out["single_env_run_eval_s"] = sorted(ts)[2]
    out["single_env_env_steps_per_s"] = len(tr.events) / out["single_env_run_eval_s"]
    for name, net in (("trained", trained), ("random", rand)):
        ro = GreedyRollout(tiers, rw, len(rates), 10000, enc, estimator_mode="true-rate", want_realized=False)
        o, ms = timed_rollout(ro, tb, net)
        red = reduce_eval(tb, o.flags, o.reward, TH, len(rates))
        t = red.totals()
        out[name] = dict(batch_ms=ms, env_steps_per_s=len(rates) * 10000 / (ms / 1e3),
                         availability_by_rate=dict(zip([str(r) for r in rates], t["availability"])),
                         mean_reward_by_rate=dict(zip([str(r) for r in rates], t["mean_reward"])))
    return out


def config2(E=4096):
    tiers = default_tiers()
    rw = RewardSpec(tasks=(TaskSpec("hellaswag", 40.0, "hard"), TaskSpec("copa", 40.0, "soft"),
                           TaskSpec("piqa", 40.0, "hard"), TaskSpec("openbookqa", 40.0, "soft")),
                    matrix=DEFAULT_MATRIX)
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    tb = TraceBatch.generate("unpredictable-time", E, 4, seed=202, n_requests=10000)
    ro = GreedyRollout(tiers, rw, E, 10000, enc, estimator_mode="estimated", want_realized=False)
    o, ms = timed_rollout(ro, tb, load_checkpoint(POL))
    red = reduce_eval(tb, o.flags, o.reward, TH, 1)
    return dict(envs=E, ms=ms, env_steps_per_s=E * 10000 / (ms / 1e3), **stats(red))


def config3():
    cfg = TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=5000,
                      log_every=5000, seed=11)
    run_training(default_tiers(), RewardSpec.default(),
                 TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=50,
                             log_every=50, seed=11), n_envs=4096, mode="graph")
    t = {}
    res = run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, timing=t, mode="graph")
    s = t["loop_ms"] / 1e3
    return dict(iterations_per_s=5000 / s, updates_per_s=res.updates / s, env_steps_per_s=4096 * 5000 / s,
                final_loss=res.log[-1].loss, transitions=res.transitions)


def config5(E=65536):
    tiers = default_tiers()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    net = load_checkpoint(POL)
    out = {}
    for name in ("unpredictable-1", "unpredictable-2", "single-task-0", "single-task-1", "single-task-2",
                 "single-task-3", "hellaswag-copa-soft"):
        sc = scenario_suite(name)
        rw = sc.adjust_rewards(RewardSpec.default())
        kw = dict(ld=10000, truncate=True) if sc.workload == "stable" else {}
        tb = TraceBatch.from_scenario(sc, E, 4, seed=505, **kw)
        ro = GreedyRollout(tiers, rw, E, tb.ld, enc, estimator_mode=sc.estimator_mode,
                           reset_between_segments=sc.reset_between_segments, want_realized=False)
        o, ms = timed_rollout(ro, tb, net, reps=2)
        red = reduce_eval(tb, o.flags, o.reward, TH, 1)
        n = int(tb.n_events.sum()) if tb.n_events is not None else E * tb.ld
        out[name] = dict(ms=ms, env_steps_per_s=n / (ms / 1e3), **stats(red))
        del ro, tb, o
        torch.cuda.empty_cache()
    return out


def main():
    torch.cuda.set_device(0)
    res = {}
    for name, fn in (("config1", config1), ("config2", config2), ("config3", config3), ("config5", config5)):
        t0 = time.time()
        res[name] = fn()
        res[name]["wall_s"] = time.time() - t0
        print(name, json.dumps(res[name])[:300], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
