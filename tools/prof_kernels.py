"""Run one rollout + one reducer launch at bench shape (for ncu -k filters)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch,
                                   default_tiers, load_checkpoint, reduce_eval)
E = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
tiers = default_tiers()
enc = StateEncoding(4, (128.0, 32.0, 8.0))
net = load_checkpoint(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/trained_seed7.beqn"))
tb = TraceBatch.generate_stable([3.0 * (1 + k % 10) for k in range(E)], N, 4, 2401, buckets=[k % 10 for k in range(E)])
ro = GreedyRollout(tiers, RewardSpec.default(), E, N, enc, estimator_mode="true-rate", want_realized=False)
for _ in range(reps):
    o = ro.launch(tb, net)
    red = reduce_eval(tb, o.flags, o.reward, (1.0, .98, .96, .94, .90), 10)
torch.cuda.synchronize()
ro.env.check()
print("ok", red.totals()["window_fraction"])
