"""Train router policies under BASELINE config 3 (4096 lockstep envs, 1M-slot
device replay, batch 512, one update per iteration = per 4096 env-steps,
200k iterations) and compare their peak-performance fractions with the four
reference-trained policies (tests/golden/trained_seed{7..10}.beqn) on the
eight reference unpredictable-1 traces.  Writes gpurun_out/config3_policies.json
(copied to profiles/ per round) and tests/golden/gpu_c3_seed<s>.beqn.

usage (GPU box): python tools/train_config3_policies.py [--iterations N] [seeds...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import policy_stats as ps  # noqa: E402
from paper_2401_07886_b200 import load_checkpoint, save_checkpoint  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=ps.CONFIG3["iterations"])
    ap.add_argument("--no-save", action="store_true")
    ap.add_argument("seeds", nargs="*", type=int)
    a = ap.parse_args()
    seeds = a.seeds or list(ps.SEEDS)
    dev = torch.device("cuda", 0)
    z = ps.traces()
    ref = {s: ps.window_fractions_gpu(load_checkpoint(os.path.join(ps.GOLDEN, f"trained_seed{s}.beqn")), z, dev)
           for s in ps.SEEDS}
    out = dict(recipe=dict(ps.CONFIG3, iterations=a.iterations), thetas=ps.THETAS,
               reference={s: v.tolist() for s, v in ref.items()}, gpu={}, train={})
    for s in seeds:
        t = {}
        t0 = time.time()
        res = ps.train_config3(s, dev, a.iterations, timing=t)
        wall = time.time() - t0
        f = ps.window_fractions_gpu(res.net, z, dev)
        out["gpu"][s] = f.tolist()
        out["train"][s] = dict(loop_s=t["loop_ms"] / 1e3, wall_s=wall, updates=res.updates,
                               transitions=res.transitions, max_inflight=res.max_inflight,
                               iterations_per_s=a.iterations / (t["loop_ms"] / 1e3),
                               final_loss=res.log[-1].loss if res.log else None)
        if not a.no_save:
            save_checkpoint(res.net, os.path.join(ps.GOLDEN, f"gpu_c3_seed{s}.beqn"))
        print(json.dumps({s: dict(fractions=f.round(4).tolist(), **out["train"][s])}), flush=True)
    ok, diff, se = ps.welch_ok(list(ref.values()), list(out["gpu"].values()))
    out["verdict"] = dict(ok=ok.tolist(), diff=diff.tolist(), two_se=(2 * se).tolist(), slack=0.02,
                          reference_mean=np.mean(list(ref.values()), axis=0).tolist(),
                          gpu_mean=np.mean(list(out["gpu"].values()), axis=0).tolist())
    print(json.dumps(out["verdict"]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "config3_policies.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
