"""Diagnose CUDA-graph replay timing of the training iteration: capture cost and
per-replay device time (events around each replay)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_07886_b200 import default_tiers, RewardSpec
import paper_2401_07886_b200.trainer as tr

orig_replay = torch.cuda.CUDAGraph.replay
times = []
def replay(self):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); orig_replay(self); e.record(); times.append((s, e))
torch.cuda.CUDAGraph.replay = replay
orig_cg = torch.cuda.graph
cap = []
class timed_graph(orig_cg):
    def __enter__(self):
        self._t0 = time.perf_counter(); return super().__enter__()
    def __exit__(self, *a):
        r = super().__exit__(*a); cap.append(time.perf_counter() - self._t0); return r
torch.cuda.graph = timed_graph
for rep in range(3):
    times.clear(); cap.clear()
    cfg = tr.TrainConfig(batch_size=512, buffer_capacity=1 << 20, warmup=10_000, total_iterations=3000,
                         log_every=3000, seed=3)
    t = {}
    tr.run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=4096, mode="graph", timing=t)
    torch.cuda.synchronize()
    per = [s.elapsed_time(e) for s, e in times]
    print(f"rep{rep}: loop {t['loop_ms']:.1f} ms, capture {sum(cap)*1e3:.1f} ms host, replays {len(per)}: "
          f"min {min(per):.2f} med {sorted(per)[len(per)//2]:.2f} max {max(per):.2f} ms, sum {sum(per):.1f}", flush=True)
