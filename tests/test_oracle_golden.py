"""Pin the CPU oracle (test infrastructure) against fixtures produced by the
reference itself (tests/golden/make_golden.py) and against the reference's
own known-answer tests (pkg/tests/test_simcore.py, test_evalkit.py)."""
import numpy as np
import pytest

import goldens
from helpers import first_diff, oracle_run
from oracle import oracle

NAMES = goldens.names()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_records(name):
    g = goldens.load(name)
    out = oracle_run(g)
    # routing decisions, queue lengths (obs), rate signal, rewards: bit-exact
    for k in ("tier", "reward", "realized", "obs", "rate"):
        i = first_diff(out[k].reshape(len(g[k]), -1).tolist() if k == "obs" else out[k],
                       g[k].tolist() if k == "obs" else g[k])
        assert np.array_equal(out[k], g[k]), f"{k} differs first at {i}"
    if out["q"] is not None:
        # OpenBLAS summation order is not reproducible: Q within 1e-9 abs
        assert np.nanmax(np.abs(out["q"] - g["q"])) < 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reducer_matches_reference(name):
    g = goldens.load(name)
    m = g["meta"]
    w = oracle.windowed(g["reward"])
    assert np.array_equal(w, g["windowed"])
    assert oracle.threshold_counts(w, m["thresholds"]) == m["counts"]
    rates = np.empty(len(g["arrival"]))
    starts = list(g["seg_start"]) + [len(rates)]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    dl = [t["deadline"] for t in m["reward"]["tasks"]]
    miss = oracle.miss_fractions_by_rate(g["realized"], g["task"], rates, dl)
    assert sorted(miss.items()) == [tuple(x) for x in m["miss_by_rate"]]


def _one_tier(alpha, beta, max_batch, tokens, replicas=1):
    return [dict(replicas=replicas, alpha_ms=alpha, beta_ms=beta, max_batch=max_batch,
                 tokens_per_request=tokens)]


HARD40 = dict(tasks=[dict(deadline=40.0, kind="hard")], matrix=[[1.0]], decay=0.01, cutoff=0.1)


def _run(tiers, arrivals, reward=HARD40):
    n = len(arrivals)
    return oracle.run_eval_oracle(tiers=tiers, reward=reward, arrival=np.array(arrivals, float),
                                  task=np.zeros(n, np.uint8), seg_start=[0], seg_rate=[1.0],
                                  forced_actions=np.zeros(n, np.uint8))


def test_known_single_request_five_ms_per_token():
    # pkg/tests/test_simcore.py:73-79: 100 tokens at alpha 4.75 + beta 0.25 -> 500 ms, 5 ms/token
    out = _run(_one_tier(4.75, 0.25, 128, 100), [0.0])
    assert out["realized"][0] == pytest.approx(5.0)


def test_known_two_simultaneous_share_batch():
    # test_simcore.py:85-95: two requests share every iteration -> 400 ms, 40 ms/token
    out = _run(_one_tier(32.0, 4.0, 8, 10), [0.0, 0.0])
    assert out["realized"] == pytest.approx([40.0, 40.0])


def test_known_queue_wait_counts():
    # test_simcore.py:109-118: max_batch 1, second request waits -> 200 ms, 20 ms/token
    out = _run(_one_tier(10.0, 0.0, 1, 10), [0.0, 0.0])
    assert out["realized"] == pytest.approx([10.0, 20.0])


def test_known_completion_at_horizon_counts():
    # test_simcore.py:103-107 / observe after 99 ms (:132-139): an END exactly at the
    # arrival is processed before the arrival observes the cluster
    out = _run(_one_tier(4.75, 0.25, 128, 100), [0.0, 500.0])
    assert out["obs"][1, 0] == 0
    out = _run(_one_tier(10.0, 0.0, 2, 5), [0.0, 0.0, 0.0, 0.0, 0.0, 99.0])
    assert out["obs"][5, 0] == 3


def test_known_min_batch_tie_breaks_low_index():
    # test_simcore.py:24-36: replicas with equal load -> lowest index first
    tiers = _one_tier(4.75, 0.25, 8, 100, replicas=4)
    out = _run(tiers, [0.0] * 6)
    assert list(out["obs"][:, 0]) == [0, 1, 2, 3, 4, 5]


def test_known_reward_soft_boundaries():
    # test_reward.py: soft 42 -> 0.98, 44 -> 0.96, 44.01 -> 0 (deadline 40, cutoff 10%)
    soft = dict(tasks=[dict(deadline=40.0, kind="soft")], matrix=[[1.0]], decay=0.01, cutoff=0.1)
    for tokens_ms, want in ((42.0, 0.98), (44.0, 0.96), (44.01, 0.0), (40.0, 1.0)):
        out = _run(_one_tier(tokens_ms, 0.0, 1, 1), [0.0], reward=soft)
        assert out["reward"][0] == pytest.approx(want, abs=1e-12)


def test_windowed_known_values():
    # test_evalkit.py:34-56
    assert np.allclose(oracle.windowed(np.ones(30)), 1.0)
    assert oracle.windowed(np.ones(5)).size == 0
    v = np.random.default_rng(0).random(100)
    naive = np.array([v[k:k + 20].mean() for k in range(81)])
    assert np.allclose(oracle.windowed(v), naive)


LEARNER_CASES = [("huber", "adam"), ("squared", "adam"), ("huber", "sgd")]


def _split(flat, like):
    out, k = {}, 0
    for name in ("w1", "b1", "w2", "b2"):
        n = like[name].size
        out[name] = flat[k:k + n].reshape(like[name].shape)
        k += n
    return out


@pytest.mark.parametrize("loss,opt", LEARNER_CASES)
def test_oracle_learner_matches_reference_train_step(loss, opt):
    """oracle.learner_step vs the reference train_step (trainer.py:276-290) on the
    recorded batches: loss, gradients, parameters and target sync."""
    gl = goldens.learner(loss, opt)
    m = gl["meta"]
    s, a, r, s2, c = goldens.replay_transitions()
    net = goldens.nets()["trained"]
    params = {k: np.array(net[k], dtype=np.float64) for k in ("w1", "b1", "w2", "b2")}
    target = {k: v.copy() for k, v in params.items()}
    adam = oracle.adam_init(params)
    flat = lambda d: np.concatenate([d[k].ravel() for k in ("w1", "b1", "w2", "b2")])
    for step in range(1, m["steps"] + 1):
        idx = gl["idx"][step - 1]
        batch = (s[idx], a[idx], r[idx], s2[idx], c[idx])
        lv, grads, new = oracle.learner_step(params, target, batch, discount=m["discount"],
                                             adam_state=adam, lr=m["lr"], loss=loss)
        if opt == "sgd":
            new = {k: params[k] - m["lr"] * grads[k] for k in params}
        assert abs(lv - gl["loss"][step - 1]) <= 1e-12 * abs(gl["loss"][step - 1])
        g_ref = gl["grad"][step - 1]
        assert np.linalg.norm(flat(grads) - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
        p_ref = gl["params"][step - 1]
        assert np.max(np.abs(flat(new) - p_ref)) <= 1e-14 + 1e-12 * np.max(np.abs(p_ref))
        params = _split(p_ref, params)  # continue from the reference's own parameters
        if step % m["target_sync_every"] == 0:
            target = {k: v.copy() for k, v in params.items()}
        assert np.array_equal(flat(target), gl["target"][step - 1])
