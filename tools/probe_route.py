"""Router throughput: fp64 router (be_qnet_route_f64) vs the tensor-core router
(be_qnet_route_tc) on B encoded states of the trained policy; CUDA events,
warm, inputs resident.  usage: python tools/probe_route.py [B] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2401_07886_b200 import TensorCoreRouter, load_checkpoint, route

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def states(B, seed=0, T=4, M=3):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.zeros((B, T + M + 1), dtype=torch.float64, device="cuda")
    x[torch.arange(B, device="cuda"), torch.randint(0, T, (B,), device="cuda", generator=g)] = 1.0
    for m, s in enumerate((128.0, 32.0, 8.0)):
        x[:, T + m] = torch.randint(0, int(2 * s), (B,), device="cuda", generator=g).double() / s
    x[:, -1] = torch.rand(B, device="cuda", generator=g, dtype=torch.float64) * (30.0 / 48.0)
    return x


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    net = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn"))
    x = states(B)
    tc = TensorCoreRouter(net, x.device)
    a_tc = torch.empty(B, dtype=torch.uint8, device="cuda")
    ms64 = timed(lambda: route(net, x, want_q=False), reps)
    ms_tc = timed(lambda: tc(x, want_q=False, out=a_tc, check=False), reps)
    tc.fallback_stats(reset=True)
    _, a_tc = tc(x, want_q=False)
    n, fb = tc.fallback_stats()
    _, a64 = route(net, x, want_q=False)
    same = bool(torch.equal(a_tc, a64))
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    byt = B * (x.shape[1] * 8 + 1)  # fp64 states in, u8 actions out
    print(json.dumps(dict(states=B, fp64_ms=ms64, tc_ms=ms_tc, fp64_states_per_s=B / ms64 * 1e3,
                          tc_states_per_s=B / ms_tc * 1e3, tc_gbs=byt / ms_tc / 1e6, hbm_frac=byt / ms_tc / 1e6 / hbm,
                          fallback_frac=fb / max(n, 1), actions_identical=same)))


if __name__ == "__main__":
    main()
