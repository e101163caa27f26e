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
