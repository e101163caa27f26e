"""Fixture generator: the reference's secondary evaluation reducers on golden runs.

Test infrastructure only.  Rebuilds reference `EvalRun`
objects (pkg/src/besteffort/evalkit.py:37-74) from the committed golden
records (tests/golden/run_*.npz, themselves produced by the reference's
run_eval) and records the UNMODIFIED reference outputs of
  selection_distribution (evalkit.py:244-262) over STABLE_SWEEP_RATES buckets,
  riemann_usage          (evalkit.py:265-270) for every (task, tier),
  collapse_rate          (evalkit.py:291-297) of miss_fractions_by_rate,
  hardware_utility       (evalkit.py:273-277),
  trial_band             (evalkit.py:280-288) over windowed series of three
                         runs on the same trace (static:0/1/2),
  running_average        (evalkit.py:212-214).
Output: tests/golden/evalstats.npz.  Usage:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_evalstats_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))

from besteffort import evalkit as ek  # noqa: E402
from besteffort.reward import RewardSpec, TaskSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = ["stable_trained", "unpredictable-1_trained", "single-task-0_trained", "stable_static1",
        "unpredictable-1_static0", "unpredictable-1_static1", "unpredictable-1_static2"]


def load(name):
    z = np.load(os.path.join(HERE, f"run_{name}.npz"))
    d = {k: z[k] for k in z.files if k != "meta"}
    d["meta"] = json.loads(str(z["meta"]))
    return d


def eval_run(g):
    n = len(g["arrival"])
    rates = np.empty(n)
    starts = list(g["seg_start"]) + [n]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    recs = [ek.RequestRecord(i, float(g["arrival"][i]), int(g["task"][i]), int(g["tier"][i]),
                             float(g["reward"][i]), float(g["realized"][i]), float(rates[i]))
            for i in range(n)]
    return ek.EvalRun(recs, "golden", 4, 0)


def spec_of(meta):
    r = meta["reward"]
    return RewardSpec(tasks=tuple(TaskSpec(t["name"], t["deadline"], t["kind"]) for t in r["tasks"]),
                      matrix=tuple(tuple(x) for x in r["matrix"]), decay_per_ms=r["decay"],
                      cutoff_fraction=r["cutoff"])


def main():
    out = {}
    buckets = np.array(ek.STABLE_SWEEP_RATES)
    for name in RUNS:
        g = load(name)
        run = eval_run(g)
        spec = spec_of(g["meta"])
        T, M = len(spec.tasks), len(spec.matrix[0])
        freq = ek.selection_distribution([run], buckets, T, M)
        out[f"{name}__freq"] = freq
        out[f"{name}__riemann"] = np.array([[ek.riemann_usage(freq, buckets, t, m) for m in range(M)]
                                            for t in range(T)])
        miss = run.miss_fractions_by_rate(spec)
        rates = sorted(miss)
        c = ek.collapse_rate(miss, rates)
        out[f"{name}__collapse"] = np.array(np.nan if c is None else c)
        out[f"{name}__hwutil"] = ek.hardware_utility(run, 8)
        out[f"{name}__running"] = ek.running_average(run.rewards())
    series = [ek.windowed(eval_run(load(f"unpredictable-1_static{k}")).rewards()) for k in range(3)]
    mean, std = ek.trial_band(series)
    out["band_mean"], out["band_std"] = mean, std
    np.savez_compressed(os.path.join(HERE, "evalstats.npz"), runs=np.array(RUNS),
                        buckets=buckets, numpy=np.array(np.__version__), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
