"""Quick throughput probe (development aid, not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import goldens
from paper_2401_07886_b200 import GreedyRollout, QNetwork, TraceBatch, default_tiers, RewardSpec, StateEncoding, reduce_eval

E = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
netname = sys.argv[3] if len(sys.argv) > 3 else "mixed1"
tiers = default_tiers()
rw = RewardSpec.default()
enc = StateEncoding(4, (128.0, 32.0, 8.0))
rates = [3.0 * (1 + (k % 10)) for k in range(E)]
tb = TraceBatch.generate_stable(rates, N, 4, seed=1234, buckets=[k % 10 for k in range(E)])
net = QNetwork.from_any(goldens.nets()[netname]) if netname != "static" else None
for skip in (True, False):
    ro = GreedyRollout(tiers, rw, E, N, enc, estimator_mode="true-rate", skip_ahead=skip, want_realized=False, ring_capacity=1024)
    for it in range(3):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        o = ro.launch(tb, net, static_tier=-1 if net is not None else 2)
        t1.record(); torch.cuda.synchronize()
        ro.env.check()
        ms = t0.elapsed_time(t1)
        print(f"skip={skip} it={it} E={E} N={N}: {ms:.2f} ms  {E*N/ms*1e3:.3e} env-steps/s", flush=True)
    mix = torch.bincount(o.tier.flatten().long(), minlength=3).tolist()
    print("tier mix", mix, "mean reward", float(o.reward.mean()))
    t0.record()
    red = reduce_eval(tb, o.flags, o.reward, thresholds=(1.0, .98, .96, .94, .90), n_buckets=10)
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    print(f"reduce: {ms:.3f} ms  {E*N*9/ms/1e6:.1f} GB/s")
    print(red.totals())
    del ro
