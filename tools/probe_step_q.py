"""How much of the step API's time is the Q forward: be_env_step with the
trained policy (fp64 qnet_group in-kernel) vs a static tier (no Q), and the
batched routers alone on the same number of states.  Device time per call,
CUDA events, after warm-up.  usage: python tools/probe_step_q.py [E ...]"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_07886_b200 import (DeviceQNet, EnvBatch, RewardSpec, StateEncoding, StepRecords,  # noqa: E402
                                   TensorCoreRouter, default_tiers, load_checkpoint, route)

dev = torch.device("cuda", 0)
net = DeviceQNet(load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn")), dev)
tiers, rw = default_tiers(), RewardSpec.default()
enc = StateEncoding(4, (128.0, 32.0, 8.0))


def timed(fn, reps=50, per_graph=20):
    """Device time per call: `per_graph` calls captured in one CUDA graph (no host
    launch overhead), replayed `reps` times."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=side):
        for _ in range(per_graph):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (reps * per_graph) * 1e3  # us


for E in [int(x) for x in sys.argv[1:]] or [4096, 16384, 65536]:
    env = EnvBatch(tiers, rw, E, enc, estimator_mode="true-rate", ring_capacity=1024)
    rec = StepRecords(E, 4096, dev, want_realized=False)
    t = torch.zeros(E, dtype=torch.float64, device=dev)
    task = torch.randint(0, 4, (E,), device=dev, dtype=torch.uint8)
    rate = torch.full((E,), 12.0, dtype=torch.float64, device=dev)

    def step(policy=None, static=-1):
        t.add_(80.0)
        env.step(t, task, rec, true_rate=rate, policy=policy, static_tier=static, want_x=True)

    us_q = timed(lambda: step(policy=net))
    us_s = timed(lambda: step(static=1))
    x = env.step(t, task, rec, true_rate=rate, policy=net, want_x=True)["x"].contiguous()
    tc = TensorCoreRouter(net.to_host(), dev)
    a = torch.empty(E, dtype=torch.uint8, device=dev)
    us_tc = timed(lambda: tc(x, want_q=False, out=a, check=False))
    from paper_2401_07886_b200 import _lib
    L = _lib.load()
    W = net.weights()
    a64 = torch.empty(E, dtype=torch.uint8, device=dev)
    us_64 = timed(lambda: _lib.check(L.be_qnet_route_f64(ctypes.byref(W), 4, 3, x.data_ptr(), E, 0.0, 0, 0, None,
                                                         a64.data_ptr(), _lib.stream_ptr())))
    print(json.dumps(dict(E=E, step_policy_us=us_q, step_static_us=us_s, q_in_step_us=us_q - us_s,
                          router_tc_us=us_tc, router_f64_us=us_64)), flush=True)
    env.close()
