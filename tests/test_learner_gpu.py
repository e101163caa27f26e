"""Device learner (be_learner_*) vs the oracle restatement of the reference
update (trainer.py:166-290): Double-Q targets, Huber loss, backward, Adam and the
target sync — fp64, so loss/grads/params agree to ~1e-12 (tolerances below).
Replay commits vs the deferred-reward rule (trainer.py:140-156)."""
import numpy as np
import pytest
import torch

import goldens
from helpers import enc_of, reward_of, tiers_of
from oracle import oracle
from paper_2401_07886_b200 import EnvBatch, QNetwork, default_tiers, RewardSpec, StateEncoding
from paper_2401_07886_b200.trainer import DeviceLearner, TrainConfig, run_training, _PendingRecords, _env_step

pytestmark = pytest.mark.gpu


def transitions_from_golden(name="unpredictable-1_trained"):
    """(s, a, r, s', cont) from a reference rollout, encoded as policy.py:52-65."""
    g = goldens.load(name)
    m = g["meta"]
    T = len(m["reward"]["tasks"])
    scales = np.array(m["enc"]["batch_scales"])
    n = len(g["arrival"])
    x = np.zeros((n, T + 3 + 1))
    x[np.arange(n), g["task"]] = 1.0
    x[:, T:T + 3] = g["obs"] / scales
    x[:, -1] = g["rate"] / m["enc"]["rate_scale"]
    return x[:-1], g["tier"][:-1], g["reward"][:-1], x[1:], np.ones(n - 1)


def params_of(net):
    get = net.__getitem__ if isinstance(net, dict) else lambda k: getattr(net, k)
    return {k: np.array(get(k), dtype=np.float64) for k in ("w1", "b1", "w2", "b2")}


def flat(d):
    return np.concatenate([d[k].ravel() for k in ("w1", "b1", "w2", "b2")])


@pytest.mark.parametrize("loss,opt", [("huber", "adam"), ("squared", "adam"), ("huber", "sgd")])
def test_learner_matches_oracle(cuda, loss, opt):
    s, a, r, s2, c = transitions_from_golden()
    B = 512
    cfg = TrainConfig(batch_size=B, buffer_capacity=4096, learning_rate=1e-3, loss=loss,
                      optimizer=opt, target_sync_every=2, warmup=0)
    L = DeviceLearner(4, 3, cfg, n_envs=1, pending_capacity=16)
    net = goldens.nets()["trained"]
    L.set_params(net)
    params = params_of(net)
    target = params_of(net)
    adam = oracle.adam_init(params)
    rng = np.random.default_rng(3)
    for step in range(1, 5):
        idx = rng.integers(0, len(a), B)
        batch = (s[idx], a[idx], r[idx], s2[idx], c[idx])
        L.backward_batch(*batch)
        L.apply(explicit_batch=True)
        if opt == "adam":
            lv, grads, new = oracle.learner_step(params, target, batch, discount=cfg.discount,
                                                 adam_state=adam, lr=cfg.learning_rate, loss=loss)
        else:
            lv, grads, _ = oracle.learner_step(params, target, batch, discount=cfg.discount,
                                               adam_state=oracle.adam_init(params),
                                               lr=cfg.learning_rate, loss=loss)
            new = {k: params[k] - cfg.learning_rate * grads[k] for k in params}
        torch.cuda.synchronize()
        g_dev = L.grad.cpu().numpy()
        g_ref = flat(grads)
        assert abs(float(L.loss[0]) - lv) <= 1e-12 * max(1.0, abs(lv))
        assert np.linalg.norm(g_dev - g_ref) <= 1e-10 * np.linalg.norm(g_ref)
        p_dev = L.params.cpu().numpy()
        p_ref = flat(new)
        assert np.max(np.abs(p_dev - p_ref)) <= 1e-12 + 1e-10 * np.max(np.abs(p_ref))
        params = new
        if step % cfg.target_sync_every == 0:  # trainer.py:288-289
            target = {k: v.copy() for k, v in params.items()}
        assert np.max(np.abs(flat(params_of(L.target_net())) - flat(target))) <= 1e-12 * 100


def test_replay_commits_follow_deferred_reward_rule(cuda):
    """Every transition (x_j, a_j, r_j, x_{j+1}) enters the ring exactly when both
    its reward and the next decision exist (trainer.py:140-156), once."""
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, (128.0, 32.0, 8.0))
    E, steps, P = 5, 300, 512
    cfg = TrainConfig(batch_size=8, buffer_capacity=100_000, warmup=10**9, total_iterations=steps)
    L = DeviceLearner(4, 3, cfg, n_envs=E, pending_capacity=P)
    net = QNetwork.from_any(goldens.nets()["mixed1"])
    L.set_params(net)
    env = EnvBatch(tiers, rw, E, enc, estimator_mode="true-rate", ring_capacity=1024)
    rec = _PendingRecords(L)
    arrival = torch.empty(E, dtype=torch.float64, device=cuda)
    task = torch.empty(E, dtype=torch.uint8, device=cuda)
    rate = torch.empty(E, dtype=torch.float64, device=cuda)
    W = L.online_weights()
    xs, acts, done_at = [], [], {}
    expected = 0
    for it in range(steps):
        L.workload(5, it, arrival, task, rate)
        slot = it % P
        _env_step(env, arrival, task, rate, W, 0.3, 9, it, rec, L.pending_x[slot], L.pending_action[slot])
        xs.append(L.pending_x[slot].clone())
        acts.append(L.pending_action[slot].clone())
        L.commit(it)
        torch.cuda.synchronize()
    L.check()
    env.check()
    size = L.size
    ring_s = L.ring_states[:size].cpu().numpy()
    ring_s2 = L.ring_next_states[:size].cpu().numpy()
    ring_a = L.ring_actions[:size].cpu().numpy()
    ring_r = L.ring_rewards[:size].cpu().numpy()
    X = torch.stack(xs).cpu().numpy()      # [steps][E][D]
    A = torch.stack(acts).cpu().numpy()
    flags = L.pending_flags.cpu().numpy()  # [E][P]
    rewards = L.pending_reward.cpu().numpy()
    # expected: every j <= steps-2 whose request has completed (flag 0x40 or committed 0x20)
    want = []
    for e in range(E):
        for j in range(steps - 1):
            f = flags[e, j % P]
            if f & 0x60:
                want.append((e, j))
    assert size == len(want)
    got = {(tuple(ring_s[k]), tuple(ring_s2[k]), int(ring_a[k])) for k in range(size)}
    for e, j in want:
        assert (tuple(X[j, e]), tuple(X[j + 1, e]), int(A[j, e])) in got
    assert np.all((ring_r >= 0) & (ring_r <= 1))


def test_run_training_smoke(cuda):
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=64, buffer_capacity=50_000, warmup=2_000, total_iterations=300,
                      log_every=100, seed=1)
    res = run_training(tiers, rw, cfg, n_envs=64)
    assert res.updates > 0
    assert res.transitions > 64 * 200
    assert len(res.log) == 3 and np.isfinite(res.log[-1].loss)
    for p in res.net.params():
        assert np.all(np.isfinite(p))


@pytest.mark.parametrize("loss,opt", [("huber", "adam"), ("squared", "adam"), ("huber", "sgd")])
def test_learner_matches_reference_golden(cuda, loss, opt):
    """Device learner vs the reference train_step's recorded I/O
    (tests/golden/make_learner_golden.py): same replay contents, same sampled
    indices -> loss (rel 1e-12), gradients (normwise 1e-10), parameters and the
    target network after every step, for six consecutive updates."""
    gl = goldens.learner(loss, opt)
    m = gl["meta"]
    s, a, r, s2, c = goldens.replay_transitions()
    cfg = TrainConfig(batch_size=m["batch"], buffer_capacity=4096, learning_rate=m["lr"], loss=loss,
                      optimizer=opt, target_sync_every=m["target_sync_every"], warmup=0)
    L = DeviceLearner(4, 3, cfg, n_envs=1, pending_capacity=16)
    L.set_params(goldens.nets()["trained"])
    for step in range(1, m["steps"] + 1):
        idx = gl["idx"][step - 1]
        L.backward_batch(s[idx], a[idx], r[idx], s2[idx], c[idx])
        L.apply(explicit_batch=True)
        torch.cuda.synchronize()
        lv = gl["loss"][step - 1]
        assert abs(float(L.loss[0]) - lv) <= 1e-12 * abs(lv)
        g_ref = gl["grad"][step - 1]
        assert np.linalg.norm(L.grad.cpu().numpy() - g_ref) <= 1e-10 * np.linalg.norm(g_ref)
        p_ref = gl["params"][step - 1]
        p_dev = L.params.cpu().numpy()
        assert np.max(np.abs(p_dev - p_ref)) <= 1e-13 + 1e-10 * np.max(np.abs(p_ref))
        t_dev = flat(params_of(L.target_net()))
        assert np.max(np.abs(t_dev - gl["target"][step - 1])) <= 1e-13 + 1e-10 * np.max(np.abs(p_ref))


def test_training_modes_bit_identical(cuda):
    """run_training through the host-driven C ABI, the device-resident
    be_train_iteration (eager) and its CUDA-graph replay give bit-identical
    networks, replay contents and logs (the graph path is the same algorithm)."""
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=64, buffer_capacity=20_000, warmup=600, total_iterations=250,
                      log_every=50, seed=5, target_sync_every=7)
    out = {}
    for mode in ("host", "device", "graph"):
        out[mode] = run_training(tiers, rw, cfg, n_envs=33, updates_per_step=2, mode=mode,
                                 graph_chunk=25)
    ref = out["host"]
    assert ref.updates > 100 and ref.transitions > 3000
    for mode in ("device", "graph"):
        r = out[mode]
        assert r.updates == ref.updates and r.transitions == ref.transitions, mode
        for a, b in zip(r.net.params(), ref.net.params()):
            assert np.array_equal(a, b), mode
        assert [(x.step, x.loss, x.mean_recent_reward, x.epsilon) for x in r.log] == \
               [(x.step, x.loss, x.mean_recent_reward, x.epsilon) for x in ref.log], mode


def test_training_modes_bit_identical_multi_round(cuda):
    """The fused env step + replay commit over more envs than one resident wave of
    CTAs (several look-back rounds per step) and a ring that wraps several times:
    the device loop still equals the host-driven loop (env step, then the separate
    commit kernel) bit for bit."""
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=128, buffer_capacity=50_000, warmup=1000, total_iterations=60,
                      log_every=20, seed=11, target_sync_every=5)
    out = {}
    for mode in ("host", "device"):
        out[mode] = run_training(tiers, rw, cfg, n_envs=6000, updates_per_step=1, mode=mode)
    ref, r = out["host"], out["device"]
    assert ref.transitions > 5 * cfg.buffer_capacity
    assert r.updates == ref.updates and r.transitions == ref.transitions and r.max_inflight == ref.max_inflight
    for a, b in zip(r.net.params(), ref.net.params()):
        assert np.array_equal(a, b)
    assert [(x.step, x.loss, x.mean_recent_reward) for x in r.log] == \
           [(x.step, x.loss, x.mean_recent_reward) for x in ref.log]


@pytest.mark.parametrize("shape", ["odd_hidden_batch", "many_replicas", "wide_hidden_big_batch"])
def test_training_fused_iteration_edge_shapes(cuda, shape):
    """The two-launch device iteration on shapes its fast paths special-case, against
    the host-driven loop (separate step, commit, tiles and update launches):
    odd_hidden_batch — hidden 100 (hidden-unit slices of unequal size, empty trailing
    slices), batch 50 (a partial last tile, fewer tiles than fused-update slices), three
    updates per iteration; many_replicas — 24 replicas per env (more than a 16-lane
    group: the step + separate commit path); wide_hidden_big_batch — batch 1024 (tiles
    that finish before the tail CTAs) and hidden 1024 (tile partials written directly,
    not staged in shared memory)."""
    rw = RewardSpec.default()
    if shape == "odd_hidden_batch":
        tiers = default_tiers()
        cfg = TrainConfig(batch_size=50, buffer_capacity=5_000, warmup=300, total_iterations=120, log_every=40,
                          seed=13, hidden=100, target_sync_every=4)
        kw = dict(n_envs=21, updates_per_step=3)
    elif shape == "many_replicas":
        tiers = default_tiers(replicas=8)
        cfg = TrainConfig(batch_size=64, buffer_capacity=5_000, warmup=300, total_iterations=120, log_every=40,
                          seed=17)
        kw = dict(n_envs=19, updates_per_step=1)
    else:  # 256 tiles (more than the fused update's tail CTAs); partials too big to stage
        tiers = default_tiers()
        cfg = TrainConfig(batch_size=1024, buffer_capacity=20_000, warmup=1_100, total_iterations=80, log_every=40,
                          seed=23, hidden=1024)
        kw = dict(n_envs=64, updates_per_step=1)
    out = {m: run_training(tiers, rw, cfg, mode=m, **kw) for m in ("host", "device", "graph")}
    ref = out["host"]
    assert ref.updates > 50
    for m in ("device", "graph"):
        r = out[m]
        assert r.updates == ref.updates and r.transitions == ref.transitions, m
        for a, b in zip(r.net.params(), ref.net.params()):
            assert np.array_equal(a, b), m
        assert [(x.step, x.loss) for x in r.log] == [(x.step, x.loss) for x in ref.log], m


@pytest.mark.parametrize("cap", ["0", "1", "5"])
def test_training_fused_commit_list_overflow(cuda, monkeypatch, cap):
    """The fused step's block transition list overflowing (BE_COMMIT_LIST_CAP shrinks
    it from 4096 entries: 0 = every transition takes the per-env overflow copy, 1 / 5 =
    an env's transitions split between the list and the overflow copy — the case a
    rescan racing the listed copies' flag updates got wrong) still fills the ring
    exactly as the host-driven loop."""
    tiers, rw = default_tiers(), RewardSpec.default()
    cfg = TrainConfig(batch_size=64, buffer_capacity=4_000, warmup=300, total_iterations=150, log_every=50,
                      seed=19)
    ref = run_training(tiers, rw, cfg, n_envs=40, updates_per_step=1, mode="host")
    monkeypatch.setenv("BE_COMMIT_LIST_CAP", cap)
    r = run_training(tiers, rw, cfg, n_envs=40, updates_per_step=1, mode="device")
    assert r.updates == ref.updates and r.transitions == ref.transitions
    for a, b in zip(r.net.params(), ref.net.params()):
        assert np.array_equal(a, b)
    assert [(x.step, x.loss, x.mean_recent_reward) for x in r.log] == \
           [(x.step, x.loss, x.mean_recent_reward) for x in ref.log]
