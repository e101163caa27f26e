"""Reducer microbenchmark (K5, be_reduce_eval): E x N synthetic rewards/flags
resident in HBM, stable single-segment traces, 5 thresholds, 10 buckets;
device time per call (CUDA events, 20 calls after 3 warm-up) and algorithmic
GB/s (9 B per request).  Library variant via BE200_LIB (A/B builds).
usage: python tools/probe_reduce.py [E] [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_07886_b200 import TraceBatch, reduce_eval  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
vals = torch.tensor([0.0, 0.45, 0.78, 1.0], dtype=torch.float64, device=dev)
reward = vals[torch.randint(0, 4, (E, N), device=dev, generator=g)]
flags = (torch.randint(0, 3, (E, N), device=dev, generator=g, dtype=torch.uint8) |
         (torch.rand((E, N), device=dev, generator=g) < 0.1).to(torch.uint8) << 7)
rates = [3.0 * (1 + e % 10) for e in range(E)]
tb = TraceBatch.generate_stable(rates, 16, 4, 7, device=dev, buckets=[e % 10 for e in range(E)])
tb.arrival = torch.empty((E, N), dtype=torch.float64, device=dev)  # reducer reads only ld/segments
tb.task = torch.empty((E, N), dtype=torch.uint8, device=dev)
th = (1.0, 0.98, 0.96, 0.94, 0.90)
for _ in range(3):
    r = reduce_eval(tb, flags, reward, th, 10)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(20):
    s.record()
    r = reduce_eval(tb, flags, reward, th, 10)
    e.record()
    torch.cuda.synchronize()
    ms.append(s.elapsed_time(e))
ms.sort()
med = ms[len(ms) // 2]
print(json.dumps(dict(lib=os.path.basename(os.environ.get("BE200_LIB", "libbe200.so")), E=E, N=N,
                      ms_median=med, ms_min=ms[0], gbs=9 * E * N / (med / 1e3) / 1e9,
                      checksum=r.totals()["win_counts"])))
