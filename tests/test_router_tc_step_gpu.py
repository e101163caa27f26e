"""The tensor-core router on the lockstep env step (north star: "tensor cores
for the batched MLP GEMMs"): the step split around a router
(be_env_step_observe -> be_qnet_route_tc -> be_env_step_submit, the reference's
own order, evalkit.py:185-205) gives the same decisions, records and states as
the fused fp64 step, and run_training(router="tc") — which routes every
iteration's E states through the certified tcgen05 router — is the same
training run bit for bit as router="fp64" in all three execution modes
(host-driven, device-resident, CUDA graph)."""
import numpy as np
import pytest
import torch

import goldens
from helpers import enc_of, reward_of, tiers_of
from paper_2401_07886_b200 import (DeviceQNet, EnvBatch, QNetwork, RewardSpec, StepRecords, TensorCoreRouter,
                                   default_tiers)
from paper_2401_07886_b200.trainer import TrainConfig, run_training

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["unpredictable-1_trained", "hellaswag-copa-soft_mixed2", "stable_trained"])
def test_observe_route_submit_equals_fused_step(cuda, name):
    """Per request: observe -> TensorCoreRouter -> submit on env A, the fused fp64
    step on env B; same encoded state, action, and (at the end) records; both
    reproduce the reference golden."""
    g = goldens.load(name)
    m = g["meta"]
    E = 5
    n = len(g["arrival"])
    net = DeviceQNet(QNetwork.from_any(goldens.net_for(m)), cuda)
    tc = TensorCoreRouter(net.to_host(), cuda)
    envs = [EnvBatch(tiers_of(m), reward_of(m), E, enc_of(m), estimator_mode=m["estimator_mode"],
                     ring_capacity=4096) for _ in range(2)]
    recs = [StepRecords(E, n, cuda) for _ in range(2)]
    arr = torch.as_tensor(np.repeat(g["arrival"][:, None], E, 1), device=cuda)
    tsk = torch.as_tensor(np.repeat(g["task"][:, None], E, 1), device=cuda)
    rates = np.empty(n)
    starts = list(g["seg_start"]) + [n]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    tr = torch.as_tensor(np.repeat(rates[:, None], E, 1), device=cuda)
    seg_starts = set(int(x) for x in g["seg_start"]) if m["reset"] else set()
    acts_a, acts_b = [], []
    for i in range(n):
        if i in seg_starts and i > 0:
            for env, rec in zip(envs, recs):
                env.new_segment(rec)
        o = envs[0].observe(arr[i], tsk[i], recs[0], true_rate=tr[i])
        _, a = tc(o["x"], want_q=False, check=False)
        envs[0].submit(arr[i], tsk[i], a, recs[0])
        ob = envs[1].step(arr[i], tsk[i], recs[1], true_rate=tr[i], policy=net, want_x=True)
        acts_a.append(a.clone())
        acts_b.append(ob["action"])
        if i % 997 == 0:
            assert torch.equal(o["x"], ob["x"]) and torch.equal(o["obs"], ob["obs"])
    for env, rec in zip(envs, recs):
        env.drain(rec)
        env.check()
    A, B = torch.stack(acts_a).cpu().numpy(), torch.stack(acts_b).cpu().numpy()
    assert np.array_equal(A, B)
    for e in range(E):
        assert np.array_equal(A[:, e], g["tier"])
    for f in ("flags", "reward", "realized"):
        assert torch.equal(getattr(recs[0], f), getattr(recs[1], f)), f
    assert np.array_equal(recs[0].reward[0].cpu().numpy(), g["reward"])


def test_submit_rejects_out_of_range_tier(cuda):
    tiers, rw = default_tiers(), RewardSpec.default()
    from paper_2401_07886_b200 import StateEncoding
    env = EnvBatch(tiers, rw, 4, StateEncoding(4, (128.0, 32.0, 8.0)), estimator_mode="true-rate",
                   ring_capacity=64)
    rec = StepRecords(4, 16, cuda)
    arr = torch.full((4,), 5.0, dtype=torch.float64, device=cuda)
    tsk = torch.zeros(4, dtype=torch.uint8, device=cuda)
    env.observe(arr, tsk, rec, true_rate=torch.full((4,), 3.0, dtype=torch.float64, device=cuda))
    env.submit(arr, tsk, torch.tensor([0, 1, 7, 2], dtype=torch.uint8, device=cuda), rec)
    with pytest.raises(ValueError):
        env.check()


@pytest.mark.parametrize("mode", ["graph", "device", "host"])
def test_training_with_tc_router_is_bit_identical(cuda, mode):
    """router="tc" vs "fp64": same networks, replay contents, logs (epsilon
    decays through exploration into greedy routing by the learning policy)."""
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=64, buffer_capacity=50_000, warmup=1_000, total_iterations=200,
                      log_every=50, seed=9, target_sync_every=13)
    out = {}
    for router in ("fp64", "tc"):
        out[router] = run_training(tiers, rw, cfg, n_envs=300, updates_per_step=2, mode=mode,
                                   graph_chunk=25, router=router)
    a, b = out["fp64"], out["tc"]
    assert a.updates > 100 and a.transitions > 20_000
    assert (a.updates, a.transitions) == (b.updates, b.transitions)
    for x, y in zip(a.net.params(), b.net.params()):
        assert np.array_equal(x, y)
    assert [(r.step, r.loss, r.mean_recent_reward) for r in a.log] == \
           [(r.step, r.loss, r.mean_recent_reward) for r in b.log]


def test_training_tc_router_rejects_unsupported_width(cuda):
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=8, buffer_capacity=64, warmup=8, total_iterations=4, hidden=48)
    with pytest.raises(ValueError):
        run_training(tiers, rw, cfg, n_envs=4, router="tc", mode="device")


def test_training_tc_router_multi_round(cuda):
    """The tensor-core step + commit over more envs than two CTAs per SM cover (several
    rounds per CTA, virtual blocks from the start-order ticket): the same training as
    the fp64 router."""
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=128, buffer_capacity=60_000, warmup=8_000, total_iterations=40, log_every=20,
                      seed=29)
    a = run_training(tiers, rw, cfg, n_envs=6000, updates_per_step=1, mode="device", router="fp64")
    b = run_training(tiers, rw, cfg, n_envs=6000, updates_per_step=1, mode="device", router="tc")
    assert a.updates > 10 and (a.updates, a.transitions) == (b.updates, b.transitions)
    for x, y in zip(a.net.params(), b.net.params()):
        assert np.array_equal(x, y)
