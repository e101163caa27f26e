"""Helpers to load the committed reference fixtures (tests/golden/*.npz)."""
import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "run_*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN, f"run_{name}.npz"))
    d = {k: z[k] for k in z.files if k != "meta"}
    d["meta"] = json.loads(str(z["meta"]))
    return d


def nets():
    out = {}
    for f in ("nets.npz", "nets_t1.npz"):
        z = np.load(os.path.join(GOLDEN, f))
        for k in z.files:
            net, p = k.rsplit("_", 1)
            out.setdefault(net, {})[p] = z[k]
    return out


def net_for(meta):
    if meta["static_tier"] >= 0:
        return None
    return nets()[meta["policy"]]


def learner(loss, opt):
    """Reference train_step I/O (tests/golden/make_learner_golden.py)."""
    z = np.load(os.path.join(GOLDEN, f"learner_{loss}_{opt}.npz"))
    d = {k: z[k] for k in z.files if k != "meta"}
    d["meta"] = json.loads(str(z["meta"]))
    return d


def replay_transitions(name="unpredictable-1_trained"):
    """(s, a, r, s', cont) of a reference rollout, encoded as policy.py:52-65 —
    the replay contents make_learner_golden.py fed the reference buffer."""
    g = load(name)
    m = g["meta"]
    T = len(m["reward"]["tasks"])
    scales = np.array(m["enc"]["batch_scales"])
    n = len(g["arrival"])
    x = np.zeros((n, T + 3 + 1))
    x[np.arange(n), g["task"]] = 1.0
    x[:, T:T + 3] = g["obs"] / scales
    x[:, -1] = g["rate"] / m["enc"]["rate_scale"]
    return x[:-1], g["tier"][:-1].astype(np.intp), g["reward"][:-1], x[1:], np.ones(n - 1)
