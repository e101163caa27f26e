"""Rollout variant choice by batch size (true rate, config-4 loads): time per launch of
each occupancy variant (0: 2 x 256-thread CTAs/SM, 128 registers; 1: 3 x 256, 80;
2: 7 x 128, 72) at several env counts (BE_ROLLOUT_FORCE_OCC), and the automatic choice.
usage: python tools/probe_occ.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch, default_tiers,  # noqa: E402
                                   load_checkpoint)

dev = torch.device("cuda", 0)
net = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn"))
enc = StateEncoding(4, (128.0, 32.0, 8.0))
N = 10000
for E in (4096, 6000, 8192, 12000, 16384, 32768):
    tb = TraceBatch.generate_stable([3.0 * (1 + g % 10) for g in range(E)], N, 4, 2401, device=dev)
    ro = GreedyRollout(default_tiers(), RewardSpec.default(), E, N, enc, estimator_mode="true-rate",
                       want_realized=False, device=dev)
    row = {"envs": E}
    for occ in ("auto", "0", "1", "2"):
        if occ == "auto":
            os.environ.pop("BE_ROLLOUT_FORCE_OCC", None)
        else:
            os.environ["BE_ROLLOUT_FORCE_OCC"] = occ
        ro.run(tb, net)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            ro.launch(tb, net)
        e.record()
        torch.cuda.synchronize()
        row[occ] = round(s.elapsed_time(e) / 3, 2)
        if occ == "auto":
            row["auto_variant"] = ro.env.rollout_plan()["throughput_variant"]
    print(json.dumps(row), flush=True)
