"""Step-synchronous env API (be_env_step / be_env_drain) vs the reference goldens:
stepping a golden trace request by request must reproduce run_eval exactly."""
import numpy as np
import pytest
import torch

import goldens
from helpers import enc_of, reward_of, tiers_of
from paper_2401_07886_b200 import EnvBatch, QNetwork, StepRecords, route

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["unpredictable-1_mixed1", "unpredictable-2_static2",
                                  "hellaswag-copa-soft_mixed2", "cfg1_32_trained_t1",
                                  "unpredictable-1_trained", "hw-utility-8gpu_trained",
                                  "stable_mixed0", "stable_trained", "stable_static1"])
def test_step_api_matches_reference(cuda, name):
    g = goldens.load(name)
    m = g["meta"]
    E = 3  # identical copies: every env must reproduce the golden
    n = len(g["arrival"])
    env = EnvBatch(tiers_of(m), reward_of(m), E, enc_of(m), estimator_mode=m["estimator_mode"],
                   ring_capacity=4096)
    rec = StepRecords(E, n, cuda)
    net = goldens.net_for(m)
    dn = QNetwork.from_any(net) if net is not None else None
    arr = torch.as_tensor(np.repeat(g["arrival"][:, None], E, 1), device=cuda)
    tsk = torch.as_tensor(np.repeat(g["task"][:, None], E, 1), device=cuda)
    rates = np.empty(n)
    starts = list(g["seg_start"]) + [n]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    tr = torch.as_tensor(np.repeat(rates[:, None], E, 1), device=cuda)
    obs, rate, act, xs = [], [], [], []
    seg_starts = set(int(x) for x in g["seg_start"]) if m["reset"] else set()
    half = torch.tensor([1, 0, 1][:E], dtype=torch.uint8, device=cuda)
    for i in range(n):
        if i in seg_starts and i > 0:
            # run_eval's segment reset (evalkit.py:186-192); masked in two calls
            env.new_segment(rec, mask=half)
            env.new_segment(rec, mask=1 - half)
        o = env.step(arr[i], tsk[i], rec, true_rate=tr[i], policy=dn, static_tier=m["static_tier"],
                     want_x=True)
        obs.append(o["obs"])
        rate.append(o["rate"])
        act.append(o["action"])
        xs.append(o["x"])
    env.drain(rec)
    env.check()
    obs = torch.stack(obs).cpu().numpy()
    rate = torch.stack(rate).cpu().numpy()
    act = torch.stack(act).cpu().numpy()
    for e in range(E):
        assert np.array_equal(obs[:, e], g["obs"])
        assert np.array_equal(rate[:, e], g["rate"])
        assert np.array_equal(act[:, e], g["tier"])
        assert np.array_equal((rec.flags[e] & 0x3F).cpu().numpy(), g["tier"])
        assert np.array_equal(rec.reward[e].cpu().numpy(), g["reward"])
        assert np.array_equal(rec.realized[e].cpu().numpy(), g["realized"])
    if dn is not None:
        # encoded states (policy.py:52-65) are exact; Q of them matches the golden
        x = torch.stack(xs)[:, 0]
        q, a = route(dn, x)
        assert np.max(np.abs(q.cpu().numpy() - g["q"])) < 1e-9
        assert np.array_equal(a.cpu().numpy(), g["tier"])


def test_epsilon_greedy_statistics(cuda):
    """select_action (policy.py:125-132): epsilon = 1 explores uniformly."""
    g = goldens.load("unpredictable-1_mixed1")
    m = g["meta"]
    E = 4096
    env = EnvBatch(tiers_of(m), reward_of(m), E, enc_of(m), ring_capacity=1024)
    rec = StepRecords(E, 64, cuda)
    arr = torch.zeros(E, dtype=torch.float64, device=cuda)
    tsk = torch.zeros(E, dtype=torch.uint8, device=cuda)
    counts = np.zeros(3)
    for i in range(8):
        arr += 1.0
        o = env.step(arr, tsk, rec, policy=QNetwork.from_any(goldens.nets()["mixed1"]),
                     epsilon=1.0, seed=11, counter=i)
        counts += np.bincount(o["action"].cpu().numpy(), minlength=3)
    p = counts / counts.sum()
    sigma = np.sqrt(1 / 3 * 2 / 3 / counts.sum())
    assert np.all(np.abs(p - 1 / 3) < 4 * sigma)
