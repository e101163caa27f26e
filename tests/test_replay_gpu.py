"""Device replay ring and training workload vs the reference semantics
(trainer.py:101-163 ReplayBuffer, :293-316 TrainingWorkload) — the GPU
analogues of the reference's own replay tests (T/test_trainer.py:63-113) plus
the sampled-index learner path against the oracle restatement of train_step.

* ring overwrite at capacity: the ring keeps the latest `capacity` commits,
  slot = commit index mod capacity (ReplayBuffer.push, trainer.py:128-139);
* uniform sampling with replacement over [0, size) (ReplayBuffer.sample,
  trainer.py:158-163; T/test_trainer.py:96 — 3 sigma per slot);
* backward on Philox-sampled ring rows == oracle.learner_step on the same rows
  (trainer.py:238-290), loss 1e-12 relative, gradients 1e-10 normwise;
* TrainingWorkload.next_arrival: log-uniform regime rates on [rate_low,
  rate_high], geometric regime lengths of mean max(1, 20 rate) (equal-time) or
  regime_mean_requests, exponential gaps of mean 1000 / rate ms, uniform tasks.
"""
import math

import numpy as np
import pytest
import torch

import goldens
from oracle import oracle
from paper_2401_07886_b200 import EnvBatch, QNetwork, RewardSpec, StateEncoding, default_tiers
from paper_2401_07886_b200.trainer import DeviceLearner, TrainConfig, _env_step, _PendingRecords

pytestmark = pytest.mark.gpu


def _fill_ring(L, s, a, r, s2, c, cursor=None):
    n = len(a)
    L.ring_states[:n].copy_(torch.as_tensor(s))
    L.ring_next_states[:n].copy_(torch.as_tensor(s2))
    L.ring_actions[:n].copy_(torch.as_tensor(np.asarray(a, np.uint8)))
    L.ring_rewards[:n].copy_(torch.as_tensor(r))
    L.ring_cont[:n].copy_(torch.as_tensor(c))
    L.ring_state[0] = (n if cursor is None else cursor) % L.cfg.buffer_capacity
    L.ring_state[1] = n
    L.ring_state[2] = n
    torch.cuda.synchronize()


def _params(net):
    return {k: np.array(getattr(net, k), np.float64) for k in ("w1", "b1", "w2", "b2")}


def _flat(d):
    return np.concatenate([d[k].ravel() for k in ("w1", "b1", "w2", "b2")])


@pytest.mark.parametrize("loss", ["huber", "squared"])
def test_sampled_backward_matches_oracle(cuda, loss):
    """Learner updates on batches the device samples from its own ring
    (be_learner_backward, Philox indices returned through sample_idx) equal the
    oracle's train_step on the rows at those indices, step after step (Adam,
    target sync every 3)."""
    s, a, r, s2, c = goldens.replay_transitions()
    n = 3000  # ring not full, not a power of two
    c = c.copy()
    c[::17] = 0.0  # a few terminal transitions (cont = 0)
    cfg = TrainConfig(batch_size=512, buffer_capacity=4096, learning_rate=1e-3, loss=loss,
                      target_sync_every=3, warmup=1000)
    L = DeviceLearner(4, 3, cfg, n_envs=1, pending_capacity=16)
    net = QNetwork.from_any(goldens.nets()["trained"])
    L.set_params(net)
    _fill_ring(L, s[:n], a[:n], r[:n], s2[:n], c[:n])
    params, target = _params(net), _params(net)
    adam = oracle.adam_init(params)
    idx = torch.empty(cfg.batch_size, dtype=torch.int64, device=cuda)
    seen = set()
    for step in range(1, 8):
        L.backward(1234, 77 + step, idx)
        L.apply()
        torch.cuda.synchronize()
        k = idx.cpu().numpy()
        assert k.min() >= 0 and k.max() < n
        seen.update(k.tolist())
        lv, grads, new = oracle.learner_step(params, target, (s[k], a[k], r[k], s2[k], c[k]),
                                             discount=cfg.discount, adam_state=adam,
                                             lr=cfg.learning_rate, loss=loss)
        assert abs(float(L.loss[0]) - lv) <= 1e-12 * abs(lv)
        g_ref = _flat(grads)
        assert np.linalg.norm(L.grad.cpu().numpy() - g_ref) <= 1e-10 * np.linalg.norm(g_ref)
        p_ref = _flat(new)
        assert np.max(np.abs(L.params.cpu().numpy() - p_ref)) <= 1e-13 + 1e-10 * np.max(np.abs(p_ref))
        params = new
        if step % cfg.target_sync_every == 0:
            target = {kk: v.copy() for kk, v in params.items()}
        t_dev = _flat(_params(L.target_net()))
        assert np.max(np.abs(t_dev - _flat(target))) <= 1e-13 + 1e-10 * np.max(np.abs(p_ref))
    assert len(seen) > 1500  # 7 x 512 draws with replacement from 3000 rows
    assert int(L.counters[1]) == 7


def test_backward_is_a_noop_during_warmup(cuda):
    """train_step returns None while len(buffer) < max(batch, warmup)
    (trainer.py:279-281): no gradient step, parameters untouched."""
    s, a, r, s2, c = goldens.replay_transitions()
    cfg = TrainConfig(batch_size=64, buffer_capacity=1024, warmup=500)
    L = DeviceLearner(4, 3, cfg, n_envs=1, pending_capacity=16)
    L.set_params(goldens.nets()["trained"])
    _fill_ring(L, s[:499], a[:499], r[:499], s2[:499], c[:499])
    p0 = L.params.clone()
    L.backward(1, 1)
    L.apply()
    torch.cuda.synchronize()
    assert int(L.counters[1]) == 0 and torch.equal(L.params, p0)
    _fill_ring(L, s[:500], a[:500], r[:500], s2[:500], c[:500])
    L.backward(1, 2)
    L.apply()
    torch.cuda.synchronize()
    assert int(L.counters[1]) == 1 and not torch.equal(L.params, p0)


@pytest.mark.parametrize("size", [8, 1000, 4096])
def test_replay_sampling_uniform_three_sigma(cuda, size):
    """rng.integers(0, size, B) analogue (trainer.py:158-163): every index in
    [0, size), each slot within 3 sigma of n/size (T/test_trainer.py:96-107 at
    size 8), a chi-square statistic within 4 sigma of its mean, and the number
    of distinct rows per batch as sampling with replacement predicts."""
    B = min(512, size)  # train_step samples only once len(buffer) >= batch
    cfg = TrainConfig(batch_size=B, buffer_capacity=size, warmup=0)
    L = DeviceLearner(4, 3, cfg, n_envs=1, pending_capacity=16)
    L.set_params(goldens.nets()["trained"])
    s, a, r, s2, c = goldens.replay_transitions()
    rows = np.arange(size) % len(a)
    _fill_ring(L, s[rows], a[rows], r[rows], s2[rows], c[rows])
    calls = max(80, 40_000 // B if size <= 16 else 160_000 // B)
    idx = torch.empty((calls, B), dtype=torch.int64, device=cuda)
    for i in range(calls):
        L.backward(99, i, idx[i])
    torch.cuda.synchronize()
    k = idx.cpu().numpy()
    assert k.min() >= 0 and k.max() < size
    n = k.size
    counts = np.bincount(k.ravel(), minlength=size)
    p = 1.0 / size
    sigma = math.sqrt(n * p * (1 - p))
    if size <= 16:
        assert np.all(np.abs(counts - n * p) < 3 * sigma), counts
    chi2 = float(((counts - n * p) ** 2 / (n * p)).sum())
    df = size - 1
    assert abs(chi2 - df) < 4 * math.sqrt(2 * df), (chi2, df)
    distinct = np.array([np.unique(row).size for row in k])
    exp_d = size * (1 - (1 - p) ** B)
    assert abs(distinct.mean() - exp_d) < 0.02 * exp_d + 1.0, (distinct.mean(), exp_d)
    # different counters draw different batches; the same counter the same batch
    L.backward(99, 0, idx[1])
    torch.cuda.synchronize()
    assert torch.equal(idx[0], idx[1])


def _commit_run(E, steps, capacity, cuda):
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, (128.0, 32.0, 8.0))
    cfg = TrainConfig(batch_size=8, buffer_capacity=capacity, warmup=10**9, total_iterations=steps)
    L = DeviceLearner(4, 3, cfg, n_envs=E, pending_capacity=512)
    L.set_params(QNetwork.from_any(goldens.nets()["mixed1"]))
    env = EnvBatch(tiers, rw, E, enc, estimator_mode="true-rate", ring_capacity=1024)
    rec = _PendingRecords(L)
    arrival = torch.empty(E, dtype=torch.float64, device=cuda)
    task = torch.empty(E, dtype=torch.uint8, device=cuda)
    rate = torch.empty(E, dtype=torch.float64, device=cuda)
    W = L.online_weights()
    for it in range(steps):
        L.workload(5, it, arrival, task, rate)
        slot = it % L.P
        _env_step(env, arrival, task, rate, W, 0.3, 9, it, rec, L.pending_x[slot], L.pending_action[slot])
        L.commit(it)
    torch.cuda.synchronize()
    L.check()
    env.check()
    out = dict(cursor=int(L.ring_state[0]), size=int(L.ring_state[1]), total=int(L.ring_state[2]),
               s=L.ring_states.cpu().numpy(), s2=L.ring_next_states.cpu().numpy(),
               a=L.ring_actions.cpu().numpy(), r=L.ring_rewards.cpu().numpy(),
               c=L.ring_cont.cpu().numpy())
    L.close()
    env.close()
    return out


def test_ring_overwrite_keeps_latest_commits(cuda):
    """The same commit stream into a ring that never wraps and one of capacity
    C that wraps several times: size == C, cursor == total mod C, and slot k of
    the small ring holds the LAST commit j with j mod C == k
    (T/test_trainer.py:89-94 at scale)."""
    E, steps, C = 7, 260, 97
    big = _commit_run(E, steps, 1 << 16, cuda)
    small = _commit_run(E, steps, C, cuda)
    total = big["total"]
    assert total == big["size"] and total > 5 * C
    assert small["total"] == total and small["size"] == C and small["cursor"] == total % C
    for k in range(C):
        j = k + ((total - 1 - k) // C) * C  # last j < total with j % C == k
        for f in ("s", "s2", "a", "r", "c"):
            assert np.array_equal(small[f][k], big[f][j]), (f, k, j)
    assert np.all(big["c"][:total] == 1.0)
    assert np.all((big["r"][:total] >= 0) & (big["r"][:total] <= 1))


def _workload_trace(cuda, E, steps, seed, **cfg_kw):
    cfg = TrainConfig(batch_size=8, buffer_capacity=64, **cfg_kw)
    L = DeviceLearner(4, 3, cfg, n_envs=E, pending_capacity=16)
    arrival = torch.empty((steps, E), dtype=torch.float64, device=cuda)
    task = torch.empty((steps, E), dtype=torch.uint8, device=cuda)
    rate = torch.empty((steps, E), dtype=torch.float64, device=cuda)
    for it in range(steps):
        L.workload(seed, it, arrival[it], task[it], rate[it])
    torch.cuda.synchronize()
    L.close()
    return arrival, task, rate


def _ks_uniform(u):
    u = np.sort(u)
    n = u.size
    i = np.arange(1, n + 1)
    return max(np.max(i / n - u), np.max(u - (i - 1) / n)) * math.sqrt(n)


def test_training_workload_rates_log_uniform(cuda):
    """Regime rate = exp(U(log rate_low, log rate_high)) (trainer.py:306-307):
    the first regime's rate of 65,536 envs passes a KS test against the
    log-uniform law (statistic < 1.63, the 1% critical value), within range."""
    E = 65536
    _, _, rate = _workload_trace(cuda, E, 1, 3)
    r = rate[0].cpu().numpy()
    lo, hi = math.log(0.25), math.log(48.0)
    assert r.min() >= 0.25 and r.max() <= 48.0
    assert _ks_uniform((np.log(r) - lo) / (hi - lo)) < 1.63
    # a different band
    _, _, rate = _workload_trace(cuda, E, 1, 4, rate_low=2.0, rate_high=8.0)
    r = rate[0].cpu().numpy()
    assert r.min() >= 2.0 and r.max() <= 8.0
    assert _ks_uniform((np.log(r) - math.log(2.0)) / (math.log(8.0) - math.log(2.0))) < 1.63


@pytest.mark.parametrize("cadence", ["equal-time", "requests"])
def test_training_workload_regimes_geometric(cuda, cadence):
    """Regime lengths (requests) are geometric(1 / mean) with mean
    max(1, regime_mean_seconds * rate) ("equal-time") or regime_mean_requests
    (trainer.py:308-312): the first regime of every env, measured in steps,
    has sum(L - mean) within 4 sigma of 0 (sigma^2 = sum (1 - p) / p^2); a
    second regime follows with a fresh rate."""
    E = 4096
    kw = dict(regime_cadence=cadence, rate_low=0.25, rate_high=8.0)
    steps = 3000 if cadence == "equal-time" else 1500
    _, _, rate = _workload_trace(cuda, E, steps, 21, **kw)
    r = rate.cpu().numpy()
    changed = r[1:] != r[:1]
    ended = changed.any(axis=0)
    first_len = np.where(ended, changed.argmax(axis=0) + 1, steps)
    r0 = r[0]
    mean = np.maximum(1.0, 20.0 * r0) if cadence == "equal-time" else np.full(E, 100.0)
    p = 1.0 / mean
    # P(L > steps) is negligible for every env (max mean 160 or 100 steps)
    assert ended.all()
    z = (first_len - mean).sum() / math.sqrt(((1 - p) / p ** 2).sum())
    assert abs(z) < 4.0, z
    # geometric's memorylessness: P(L > mean) ~= (1 - p)^mean ~ e^-1
    frac = float((first_len > mean).mean())
    exp_frac = float(((1 - p) ** np.floor(mean)).mean())
    assert abs(frac - exp_frac) < 4 * math.sqrt(exp_frac * (1 - exp_frac) / E), (frac, exp_frac)


def test_training_workload_gaps_and_tasks(cuda):
    """Gaps Exp(mean 1000 / rate) ms (trainer.py:313): gap * rate / 1000 is
    Exp(1) (KS < 1.63 on its CDF, mean and variance within 4 sigma); arrivals
    strictly increase; tasks uniform over n_tasks (3 sigma per task)."""
    E, steps = 2048, 200
    arrival, task, rate = _workload_trace(cuda, E, steps, 8)
    a = arrival.cpu().numpy()
    r = rate.cpu().numpy()
    gaps = np.diff(np.vstack([np.zeros((1, E)), a]), axis=0)
    assert np.all(gaps > 0)
    z = (gaps * r / 1000.0).ravel()
    n = z.size
    assert abs(z.mean() - 1.0) < 4 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 4 * math.sqrt(8.0 / n)
    assert _ks_uniform(1.0 - np.exp(-z[:200_000])) < 1.63
    t = task.cpu().numpy().ravel()
    counts = np.bincount(t, minlength=4)
    assert counts.size == 4
    sigma = math.sqrt(t.size * 0.25 * 0.75)
    assert np.all(np.abs(counts - t.size / 4) < 3 * sigma), counts
