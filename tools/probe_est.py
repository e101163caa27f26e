"""Estimated-rate rollout (configs 2/5: device unpredictable-1 traces, mixed deadlines)
with the latency variant (2 CTAs/SM) vs the throughput variant (3 CTAs/SM) forced
(BE_ROLLOUT_FORCE_OCC), at 4,096 and 65,536 envs."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch, default_tiers,  # noqa: E402
                                   load_checkpoint)
dev = torch.device("cuda", 0)
net = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn"))
enc = StateEncoding(4, (128.0, 32.0, 8.0))
for E in (4096, 16384, 65536):
    tb = TraceBatch.generate("unpredictable-time", E, 4, 77, n_requests=10000, device=dev)
    ro = GreedyRollout(default_tiers(), RewardSpec.default(), E, tb.ld, enc, estimator_mode="estimated",
                       want_realized=False, device=dev)
    row = {"envs": E}
    for occ in ("0", "1"):
        os.environ["BE_ROLLOUT_FORCE_OCC"] = occ
        ro.run(tb, net)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            ro.launch(tb, net)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 3
        row[occ] = dict(ms=round(ms, 2), steps_per_s=E * 10000 / ms * 1e3)
    print(json.dumps(row), flush=True)
