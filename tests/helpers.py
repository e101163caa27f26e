"""Shared test helpers: build specs from golden metadata, run the oracle."""
import numpy as np

import goldens
from oracle import oracle
from paper_2401_07886_b200 import specs


def tiers_of(meta):
    return [specs.ModelTierSpec(i, **t) for i, t in enumerate(meta["tiers"])]


def reward_of(meta):
    r = meta["reward"]
    return specs.RewardSpec(tasks=tuple(specs.TaskSpec(t["name"], t["deadline"], t["kind"])
                                        for t in r["tasks"]),
                            matrix=tuple(tuple(x) for x in r["matrix"]),
                            decay_per_ms=r["decay"], cutoff_fraction=r["cutoff"])


def enc_of(meta):
    return specs.StateEncoding(len(meta["reward"]["tasks"]), tuple(meta["enc"]["batch_scales"]),
                               meta["enc"]["rate_scale"])


def oracle_run(g, **kw):
    m = g["meta"]
    args = dict(tiers=m["tiers"], reward=m["reward"], arrival=g["arrival"], task=g["task"],
                seg_start=g["seg_start"], seg_rate=g["seg_rate"], net=goldens.net_for(m),
                static_tier=m["static_tier"], batch_scales=m["enc"]["batch_scales"],
                rate_scale=m["enc"]["rate_scale"], estimator_mode=m["estimator_mode"],
                reset=m["reset"])
    args.update(kw)
    return oracle.run_eval_oracle(**args)


def first_diff(a, b):
    d = np.nonzero(np.asarray(a) != np.asarray(b))[0]
    return int(d[0]) if d.size else -1
