"""Parity of the fused GPU rollout (be_rollout_greedy) with the reference
(golden records) and the CPU oracle.  Bit-exact: routing decisions, queue
lengths (obs), rate signal, rewards, realized latency, deadline misses.
Q-values: |dQ| <= 1e-9 (fp64; OpenBLAS order not reproducible)."""
import numpy as np
import pytest
import torch

import goldens
from helpers import enc_of, first_diff, oracle_run, reward_of, tiers_of
from paper_2401_07886_b200 import (CapacityError, GreedyRollout, QNetwork, StateEncoding, TraceBatch,
                                   reduce_eval, run_eval)
from oracle import oracle

pytestmark = pytest.mark.gpu
NAMES = goldens.names()


def gpu_run(g, skip=True, want_steps=True, n_copies=1, ring_capacity=None, forced=None):
    m = g["meta"]
    arr = np.tile(g["arrival"], (n_copies, 1))
    tsk = np.tile(g["task"], (n_copies, 1))
    ss = [list(g["seg_start"])] * n_copies
    sr = [list(g["seg_rate"])] * n_copies
    tb = TraceBatch.from_arrays(arr, tsk, ss, sr)
    ro = GreedyRollout(tiers_of(m), reward_of(m), n_copies, tb.ld, enc_of(m),
                       estimator_mode=m["estimator_mode"], reset_between_segments=m["reset"],
                       skip_ahead=skip, want_steps=want_steps, ring_capacity=ring_capacity)
    net = goldens.net_for(m)
    f = None if forced is None else torch.as_tensor(np.tile(forced, (n_copies, 1)), device="cuda")
    if f is not None:
        return ro.run(tb, forced=f), tb
    if net is None:
        return ro.run(tb, static_tier=m["static_tier"]), tb
    return ro.run(tb, QNetwork.from_any(net)), tb


def assert_env_equal(o, e, g, check_q=True):
    n = len(g["arrival"])
    tier = o.tier[e, :n].cpu().numpy()
    i = first_diff(tier, g["tier"])
    if i >= 0:
        pytest.fail(f"tier differs first at request {i} (fp64 ref margin {g['margin'][i]:.3g})")
    assert np.array_equal(o.reward[e, :n].cpu().numpy(), g["reward"])
    assert np.array_equal(o.realized[e, :n].cpu().numpy(), g["realized"])
    dl = np.array([t["deadline"] for t in g["meta"]["reward"]["tasks"]])
    miss = g["realized"] > dl[g["task"]]
    assert np.array_equal(o.miss[e, :n].cpu().numpy(), miss)
    if o.obs is not None:
        assert np.array_equal(o.obs[e, :n].cpu().numpy(), g["obs"])
        assert np.array_equal(o.rate[e, :n].cpu().numpy(), g["rate"])
        if check_q and g["meta"]["static_tier"] < 0:
            assert np.max(np.abs(o.q[e, :n].cpu().numpy() - g["q"])) < 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_rollout_matches_reference(cuda, name):
    g = goldens.load(name)
    o, _ = gpu_run(g)
    assert_env_equal(o, 0, g)


@pytest.mark.parametrize("name", [n for n in NAMES if "static" in n or "quantized" in n])
def test_rollout_without_skip_matches(cuda, name):
    g = goldens.load(name)
    o, _ = gpu_run(g, skip=False)
    assert_env_equal(o, 0, g)


@pytest.mark.parametrize("name", ["unpredictable-1_mixed2", "stable_static2", "unpredictable-2_static2"])
def test_rollout_batch_of_copies(cuda, name):
    g = goldens.load(name)
    o, _ = gpu_run(g, n_copies=257, want_steps=False)
    for e in (0, 1, 128, 256):
        assert_env_equal(o, e, g)
    t = o.tier[:, :len(g["arrival"])]
    assert bool((t == t[0:1]).all())


@pytest.mark.parametrize("scenario", ["unpredictable-1", "stable", "hellaswag-copa-soft"])
def test_ragged_batch_matches_oracle(cuda, scenario):
    """Many envs of different lengths in one launch (exercises the persistent
    env scheduler, two envs per warp and mid-warp env refills)."""
    names = [n for n in NAMES if n.startswith(scenario + "_")]
    gs = [goldens.load(n) for n in names]
    m = gs[0]["meta"]
    net = goldens.nets()["mixed1"]
    rng = np.random.default_rng(7)
    traces = []
    for k in range(61):
        g = gs[k % len(gs)]
        n = int(rng.integers(0, len(g["arrival"]) + 1))
        ss = [s for s in g["seg_start"] if s < max(n, 1)] or [0]
        traces.append((g["arrival"][:n], g["task"][:n], ss, list(g["seg_rate"][:len(ss)])))
    ld = max(len(t[0]) for t in traces)
    arr = np.zeros((len(traces), ld))
    tsk = np.zeros((len(traces), ld), np.uint8)
    for e, t in enumerate(traces):
        arr[e, :len(t[0])] = t[0]
        if len(t[0]):
            arr[e, len(t[0]):] = t[0][-1]
        tsk[e, :len(t[1])] = t[1]
    tb = TraceBatch.from_arrays(arr, tsk, [t[2] for t in traces], [t[3] for t in traces],
                                n_events=[len(t[0]) for t in traces])
    ro = GreedyRollout(tiers_of(m), reward_of(m), len(traces), ld, enc_of(m),
                       estimator_mode=m["estimator_mode"], reset_between_segments=m["reset"],
                       want_steps=True)
    o = ro.run(tb, QNetwork.from_any(net))
    for e, t in enumerate(traces):
        n = len(t[0])
        ref = oracle.run_eval_oracle(tiers=m["tiers"], reward=m["reward"], arrival=t[0], task=t[1],
                                     seg_start=t[2], seg_rate=t[3], net=net,
                                     batch_scales=m["enc"]["batch_scales"],
                                     estimator_mode=m["estimator_mode"], reset=m["reset"])
        assert np.array_equal(o.tier[e, :n].cpu().numpy(), ref["tier"]), f"env {e}"
        assert np.array_equal(o.reward[e, :n].cpu().numpy(), ref["reward"]), f"env {e}"
        assert np.array_equal(o.obs[e, :n].cpu().numpy(), ref["obs"]), f"env {e}"


def test_forced_actions_match_oracle(cuda):
    g = goldens.load("unpredictable-1_mixed1")
    forced = np.random.default_rng(1).integers(0, 3, size=len(g["arrival"])).astype(np.uint8)
    o, _ = gpu_run(g, forced=forced)
    ref = oracle_run(g, forced_actions=forced, net=None)
    assert np.array_equal(o.tier[0].cpu().numpy(), forced)
    assert np.array_equal(o.reward[0].cpu().numpy(), ref["reward"])
    assert np.array_equal(o.obs[0].cpu().numpy(), ref["obs"])


def test_ring_overflow_raises(cuda):
    g = goldens.load("unpredictable-2_static2")  # large tier floods: queues grow to ~hundreds
    with pytest.raises(CapacityError):
        gpu_run(g, ring_capacity=8, want_steps=False)


def test_run_eval_dropin_records(cuda):
    g = goldens.load("hellaswag-copa-soft_mixed0")
    m = g["meta"]
    from paper_2401_07886_b200.specs import ArrivalEvent, SegmentMark, WorkloadTrace
    tr = WorkloadTrace([ArrivalEvent(float(t), int(k)) for t, k in zip(g["arrival"], g["task"])],
                       [SegmentMark(int(a), float(b)) for a, b in zip(g["seg_start"], g["seg_rate"])], 0)
    run = run_eval(QNetwork.from_any(goldens.net_for(m)), tr, tiers_of(m), reward_of(m), enc_of(m),
                   estimator_mode=m["estimator_mode"], reset_between_segments=m["reset"])
    assert [r.tier_id for r in run.records] == g["tier"].tolist()
    assert [r.reward for r in run.records] == g["reward"].tolist()
    assert [r.realized_ms_per_token for r in run.records] == g["realized"].tolist()
    assert sorted(run.miss_fractions_by_rate(reward_of(m)).items()) == [tuple(x) for x in m["miss_by_rate"]]


@pytest.mark.parametrize("name", NAMES)
def test_reducer_matches_reference(cuda, name):
    g = goldens.load(name)
    m = g["meta"]
    o, tb = gpu_run(g, want_steps=False)
    red = reduce_eval(tb, o.flags, o.reward, thresholds=m["thresholds"])
    assert red.win_counts[0].cpu().tolist() == m["counts"]
    assert int(red.n_windows[0]) == m["n_windows"]
    dl = np.array([t["deadline"] for t in m["reward"]["tasks"]])
    assert int(red.bucket_miss[0, 0]) == int(np.sum(g["realized"] > dl[g["task"]]))
    assert int(red.bucket_req[0, 0]) == len(g["arrival"])
    assert float(red.bucket_reward[0, 0]) == pytest.approx(float(np.sum(g["reward"])), rel=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_skip_table_random_tiers_match_oracle(cuda, seed):
    """Exact iteration skipping (host-tabulated per-(tier, n, binade) increments)
    against the oracle's one-iteration-at-a-time recurrence on random,
    mostly non-dyadic tier constants (alpha in (0.1, 40), beta in {0, dyadic,
    non-dyadic}), few tokens, arrivals quantised to force END == arrival ties,
    and traces that cross many binades."""
    rng = np.random.default_rng(100 + seed)
    M = int(rng.integers(1, 4))
    tiers = []
    for m in range(M):
        beta = [0.0, 0.25, 1.2, float(rng.uniform(0.01, 3.0)), 1.0 / 3.0][int(rng.integers(0, 5))]
        tiers.append(dict(replicas=int(rng.integers(1, 5)), alpha_ms=float(rng.uniform(0.1, 40.0)),
                          beta_ms=beta, max_batch=int(rng.integers(1, 9)),
                          tokens_per_request=int(rng.integers(1, 200))))
    T = 2
    reward = dict(tasks=[dict(name="a", deadline=40.0, kind="hard"), dict(name="b", deadline=25.0, kind="soft")],
                  matrix=[[float(x) for x in rng.uniform(0, 1, M)] for _ in range(T)],
                  decay=0.01, cutoff=0.1)
    E, n = 24, 3000
    arr = np.cumsum(rng.exponential(rng.uniform(5, 400), size=(E, n)), axis=1)
    arr[::2] = np.floor(arr[::2] / 5.0) * 5.0  # quantised: ties between END and arrivals
    tsk = rng.integers(0, T, size=(E, n)).astype(np.uint8)
    forced = rng.integers(0, M, size=(E, n)).astype(np.uint8)
    meta = dict(tiers=tiers, reward=reward)
    tb = TraceBatch.from_arrays(arr, tsk, [[0]] * E, [[1.0]] * E)
    ro = GreedyRollout(tiers_of(meta), reward_of(meta), E, n, None, estimator_mode="estimated",
                       want_steps=True)
    o = ro.run(tb, forced=torch.as_tensor(forced, device=cuda))
    for e in range(E):
        ref = oracle.run_eval_oracle(tiers=tiers, reward=reward, arrival=arr[e], task=tsk[e],
                                     seg_start=[0], seg_rate=[1.0], forced_actions=forced[e])
        for k in ("reward", "realized", "obs"):
            got = getattr(o, k)[e, :n].cpu().numpy()
            assert np.array_equal(got, ref[k]), f"env {e} {k} first diff {first_diff(got.ravel(), ref[k].ravel())}"


# ---------------------------------------------------------------------------
# Certified fp32 decision screen (be_env.cuh qnet_screen): runs that do not
# record Q values decide with the screen and fall back to fp64 where it cannot
# certify; every decision must still equal the reference's.
POLICY_NAMES = [n for n in NAMES if goldens.load(n)["meta"]["static_tier"] < 0]


@pytest.mark.parametrize("name", POLICY_NAMES)
def test_screened_rollout_matches_reference(cuda, name):
    g = goldens.load(name)
    m = g["meta"]
    arr, tsk = g["arrival"][None], g["task"][None]
    tb = TraceBatch.from_arrays(arr, tsk, [list(g["seg_start"])], [list(g["seg_rate"])])
    ro = GreedyRollout(tiers_of(m), reward_of(m), 1, tb.ld, enc_of(m),
                       estimator_mode=m["estimator_mode"], reset_between_segments=m["reset"],
                       want_steps=False)
    ro.env.screen_stats(reset=True)
    o = ro.run(tb, QNetwork.from_any(goldens.net_for(m)))
    assert_env_equal(o, 0, g)
    screened, fallback = ro.env.screen_stats()
    assert screened == len(g["arrival"])
    assert 0 <= fallback <= screened


def test_screen_equals_fp64_on_large_batch(cuda):
    """Screen on vs off over many envs of device-generated traces (bench-like
    workload, trained policy): identical flags and rewards bit for bit."""
    from paper_2401_07886_b200 import RewardSpec, StateEncoding, default_tiers, load_checkpoint
    import os
    E, N = 1024, 4000
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    net = load_checkpoint(os.path.join(goldens.GOLDEN, "trained_seed7.beqn"))
    rates = [3.0 * (1 + (e % 10)) for e in range(E)]
    tb = TraceBatch.generate_stable(rates, N, 4, 11, device=cuda)
    outs = []
    for screen in (True, False):
        ro = GreedyRollout(tiers, rw, E, N, enc, estimator_mode="true-rate", want_realized=False,
                           q_screen=screen)
        ro.env.screen_stats(reset=True)
        o = ro.run(tb, net)
        outs.append((o.flags.clone(), o.reward.clone(), ro.env.screen_stats()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    screened, fallback = outs[0][2]
    assert screened == E * N and fallback < 0.1 * screened
    assert outs[1][2] == (0, 0)


def test_screen_falls_back_on_exact_ties(cuda):
    """Two actions with identical Q everywhere: the screen can never certify,
    so every decision comes from the fp64 path (first maximum, np.argmax)."""
    g = goldens.load("unpredictable-1_mixed1")
    m = g["meta"]
    net = {k: v.copy() for k, v in goldens.net_for(m).items()}
    net["w2"][:, 2] = net["w2"][:, 1]
    net["b2"][2] = net["b2"][1]
    net["b2"][1:] += 50.0  # tiers 1/2 dominate tier 0
    tb = TraceBatch.from_arrays(g["arrival"][None], g["task"][None], [list(g["seg_start"])],
                                [list(g["seg_rate"])])
    res = []
    for screen in (True, False):
        ro = GreedyRollout(tiers_of(m), reward_of(m), 1, tb.ld, enc_of(m),
                           estimator_mode=m["estimator_mode"], reset_between_segments=m["reset"],
                           want_steps=False, q_screen=screen)
        ro.env.screen_stats(reset=True)
        o = ro.run(tb, QNetwork.from_any(net))
        res.append((o.tier[0].cpu().numpy(), ro.env.screen_stats()))
    assert np.array_equal(res[0][0], res[1][0])
    assert not np.any(res[0][0] == 2)  # first maximum wins the tie
    n = len(g["arrival"])
    assert res[0][1] == (n, n)
    ref = oracle.run_eval_oracle(tiers=m["tiers"], reward=m["reward"], arrival=g["arrival"], task=g["task"],
                                 seg_start=g["seg_start"], seg_rate=g["seg_rate"], net=net,
                                 batch_scales=m["enc"]["batch_scales"],
                                 estimator_mode=m["estimator_mode"], reset=m["reset"])
    assert np.array_equal(res[0][0], ref["tier"])


@pytest.mark.parametrize("name", ["unpredictable-1_trained", "stable_mixed1", "hellaswag-copa-soft_mixed0"])
def test_wide_rings_use_unpacked_observe(cuda, name):
    """Ring capacity 1024 x 4 replicas per tier exceeds the 10-bit packed observe
    fields, so the kernel sums each tier with its own REDUX: same results."""
    g = goldens.load(name)
    o, _ = gpu_run(g, ring_capacity=1024)
    assert_env_equal(o, 0, g)


@pytest.mark.parametrize("seed", range(8))
def test_screen_random_configs_equal_fp64(cuda, seed):
    """Certified screen vs fp64 decisions on random clusters and networks: 1-8
    tiers (packed and unpacked observe), up to 24 replicas (32-lane groups),
    hidden 32-512, weights scaled up to make near-ties and large bounds common,
    estimated rates on bursty traces (huge rate inputs).  Flags and rewards must
    be identical bit for bit, whatever the fallback rate."""
    rng = np.random.default_rng(500 + seed)
    M = int(rng.choice([1, 2, 3, 4, 5, 8]))
    T = int(rng.integers(1, 5))
    H = int(rng.choice([32, 64, 128, 256, 512]))
    tiers = []
    for m in range(M):
        tiers.append(dict(replicas=int(rng.integers(1, 25 // M + 1)), alpha_ms=float(rng.uniform(0.5, 30.0)),
                          beta_ms=float(rng.uniform(0.05, 4.0)), max_batch=int(rng.integers(1, 64)),
                          tokens_per_request=int(rng.integers(5, 120))))
    reward = dict(tasks=[dict(name=f"t{t}", deadline=float(rng.uniform(5, 60)), kind=["hard", "soft"][t % 2])
                         for t in range(T)],
                  matrix=[[float(x) for x in rng.uniform(0, 1, M)] for _ in range(T)], decay=0.01, cutoff=0.1)
    meta = dict(tiers=tiers, reward=reward)
    net = QNetwork.init_random(T, M, H, rng)
    scale = float(rng.choice([1.0, 30.0, 300.0]))
    net.w2 = net.w2 * scale
    net.b1 = rng.normal(0, 0.3, H)
    net.b2 = rng.normal(0, 0.01 * scale, M)
    E, n = 96, 1500
    gaps = rng.exponential(1.0, size=(E, n)) * np.where(rng.random((E, n)) < 0.1, 0.05, 60.0)
    arr = np.cumsum(gaps, axis=1)
    tsk = rng.integers(0, T, size=(E, n)).astype(np.uint8)
    tb = TraceBatch.from_arrays(arr, tsk, [[0]] * E, [[1.0]] * E)
    enc = StateEncoding(T, tuple(float(t["max_batch"]) for t in tiers))
    outs = []
    for screen in (True, False):
        ro = GreedyRollout(tiers_of(meta), reward_of(meta), E, n, enc, estimator_mode="estimated",
                           q_screen=screen, ring_capacity=4096)
        ro.env.screen_stats(reset=True)
        o = ro.run(tb, net)
        outs.append((o.flags.clone(), o.reward.clone(), ro.env.screen_stats()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    screened, fallback = outs[0][2]
    lpe = 16 if sum(t["replicas"] for t in tiers) <= 16 else 32
    assert screened == (E * n if H % (2 * lpe) == 0 else 0)  # the screen needs H % (2 LPE) == 0
    assert 0 <= fallback <= screened
