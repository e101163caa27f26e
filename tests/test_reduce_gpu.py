"""Evaluation reducer (be_reduce_eval) vs the oracle restatement of
evalkit.windowed / threshold_counts (evalkit.py:217-241) and the per-rate
miss fractions (evalkit.py:61-68): counts bit-exact, reward sums to 1e-12."""
import os

import numpy as np
import pytest
import torch

import goldens
from oracle import oracle
from paper_2401_07886_b200 import InvalidParameterError, TraceBatch, reduce_eval

pytestmark = pytest.mark.gpu
VALUES = np.array([0.0, 0.45, 0.78, 1.0, 0.8, 0.95, 0.82, 0.96, 0.7, 0.94, 0.98, 0.96])


def make_case(E, ld, seed, ragged=True, n_buckets=3):
    rng = np.random.default_rng(seed)
    n = rng.integers(0, ld + 1, E) if ragged else np.full(E, ld)
    reward = np.zeros((E, ld))
    flags = np.zeros((E, ld), np.uint8)
    ss, sr, sb = [], [], []
    for e in range(E):
        p = rng.dirichlet(np.ones(len(VALUES)) * 0.3)
        # long runs of 1.0 make exact-peak windows (theta == 1.0) non-trivial
        r = np.where(rng.random(n[e]) < 0.7, 1.0, rng.choice(VALUES, n[e], p=p))
        reward[e, :n[e]] = r
        flags[e, :n[e]] = rng.integers(0, 3, n[e]) | ((r == 0) << 7).astype(np.uint8)
        k = int(rng.integers(1, 5))
        starts = np.sort(rng.integers(0, max(int(n[e]), 1), k))
        starts[0] = 0
        ss.append(starts.tolist())
        sr.append(rng.random(k).tolist())
        sb.append(rng.integers(0, n_buckets, k).tolist())
    return n, reward, flags, ss, sr, sb


@pytest.mark.parametrize("E,ld,ragged", [(1, 10000, False), (77, 1000, True), (1000, 333, True),
                                         (64, 4096, False), (33, 25, True),
                                         # >= one CTA of 4 warps x 2 groups per SM: the big-batch tile
                                         # shape (256-byte bursts, two 32-env groups per warp)
                                         (40000, 70, True), (38000, 96, False)])
def test_reduce_matches_oracle(cuda, E, ld, ragged):
    n, reward, flags, ss, sr, sb = make_case(E, ld, seed=E + ld, ragged=ragged)
    th = (1.0, 0.99, 0.98, 0.96, 0.94, 0.90)
    tb = TraceBatch.from_arrays(np.zeros((E, ld)), np.zeros((E, ld), np.uint8), ss, sr,
                                n_events=n if ragged else None, seg_bucket=sb)
    red = reduce_eval(tb, torch.as_tensor(flags, device="cuda"),
                      torch.as_tensor(reward, device="cuda"), thresholds=th, n_buckets=3)
    wc = red.win_counts.cpu().numpy()
    nw = red.n_windows.cpu().numpy()
    bm, bq = red.bucket_miss.cpu().numpy(), red.bucket_req.cpu().numpy()
    brw = red.bucket_reward.cpu().numpy()
    for e in range(E):
        r = reward[e, :n[e]]
        w = oracle.windowed(r)
        assert nw[e] == w.size
        assert wc[e].tolist() == oracle.threshold_counts(w, th), f"env {e}"
        bucket = np.zeros(n[e], int)
        starts = list(ss[e]) + [n[e]]
        for k in range(len(ss[e])):
            bucket[starts[k]:starts[k + 1]] = sb[e][k]
        for b in range(3):
            sel = bucket == b
            assert bq[e, b] == sel.sum()
            assert bm[e, b] == (flags[e, :n[e]][sel] >> 7).sum()
            assert brw[e, b] == pytest.approx(r[sel].sum(), rel=1e-12, abs=1e-12)


def test_reduce_rejects_bad_args(cuda):
    tb = TraceBatch.from_arrays(np.zeros((1, 30)), np.zeros((1, 30), np.uint8), [[0]], [[1.0]])
    f = torch.zeros((1, 30), dtype=torch.uint8, device="cuda")
    r = torch.zeros((1, 30), dtype=torch.float64, device="cuda")
    with pytest.raises(InvalidParameterError):
        reduce_eval(tb, f, r, thresholds=(1.5,))
    with pytest.raises(InvalidParameterError):
        reduce_eval(tb, f, r, thresholds=(0.9,), window=7)


def _evalstats():
    z = np.load(os.path.join(goldens.GOLDEN, "evalstats.npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", ["stable_trained", "unpredictable-1_trained", "single-task-0_trained",
                                  "stable_static1"])
def test_selection_and_secondary_reducers_match_reference(cuda, name):
    """selection_distribution / riemann_usage / collapse_rate / hardware_utility /
    running_average vs the reference's own outputs on the golden records
    (tests/golden/make_evalstats_golden.py); counting runs on the device."""
    from paper_2401_07886_b200.evalkit import (STABLE_SWEEP_RATES, collapse_rate, hardware_utility,
                                               riemann_usage, running_average, selection_distribution)
    ref = _evalstats()
    g = goldens.load(name)
    m = g["meta"]
    n = len(g["arrival"])
    tb = TraceBatch.from_arrays(g["arrival"], g["task"], list(g["seg_start"]), list(g["seg_rate"]))
    flags = torch.as_tensor(g["tier"].astype(np.uint8)[None, :], device=cuda)
    T, M = len(m["reward"]["tasks"]), len(m["tiers"])
    freq = selection_distribution(tb, STABLE_SWEEP_RATES, T, M, flags=flags)
    assert np.array_equal(freq, ref[f"{name}__freq"])
    rie = np.array([[riemann_usage(freq, STABLE_SWEEP_RATES, t, k) for k in range(M)] for t in range(T)])
    assert np.array_equal(rie, ref[f"{name}__riemann"])
    rates = np.empty(n)
    starts = list(g["seg_start"]) + [n]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    dl = np.array([t["deadline"] for t in m["reward"]["tasks"]])
    miss = {float(r): float(np.mean((g["realized"] > dl[g["task"]])[rates == r])) for r in np.unique(rates)}
    c = collapse_rate(miss, sorted(miss))
    want = ref[f"{name}__collapse"]
    assert (c is None and np.isnan(want)) or c == float(want)
    assert np.array_equal(hardware_utility(g["reward"], 8), ref[f"{name}__hwutil"])
    assert np.array_equal(running_average(g["reward"]), ref[f"{name}__running"])


def test_windowed_series_and_trial_band_match_reference(cuda):
    from paper_2401_07886_b200.evalkit import trial_band, windowed
    ref = _evalstats()
    gs = [goldens.load(f"unpredictable-1_static{k}") for k in range(3)]
    tb = TraceBatch.from_arrays(np.stack([g["arrival"] for g in gs]), np.stack([g["task"] for g in gs]),
                                [list(g["seg_start"]) for g in gs], [list(g["seg_rate"]) for g in gs])
    rw = torch.as_tensor(np.stack([g["reward"] for g in gs]), device=cuda)
    w = windowed(tb, rw)
    n = len(gs[0]["reward"]) - 19
    for k, g in enumerate(gs):
        assert np.array_equal(w[k, :n].cpu().numpy(), oracle.windowed(g["reward"]))
    mean, std = trial_band([w[k, :n].cpu().numpy() for k in range(3)])
    assert np.array_equal(mean, ref["band_mean"]) and np.array_equal(std, ref["band_std"])


def test_selection_counts_many_envs(cuda):
    """Ragged multi-env batch: device (task, bucket, tier) counts == numpy."""
    from paper_2401_07886_b200.evalkit import selection_counts
    rng = np.random.default_rng(4)
    E, ld, T, M, K = 77, 700, 4, 3, 5
    n = rng.integers(0, ld + 1, E)
    task = rng.integers(0, T, (E, ld)).astype(np.uint8)
    flags = (rng.integers(0, M, (E, ld)) | 0x40 | (rng.integers(0, 2, (E, ld)) << 7)).astype(np.uint8)
    ss, sr, sb = [], [], []
    want = np.zeros((T, K, M), np.int64)
    for e in range(E):
        cuts = sorted(set([0] + list(rng.integers(1, max(2, n[e]), rng.integers(0, 6)))))
        ss.append(cuts)
        sr.append([1.0] * len(cuts))
        sb.append(list(rng.integers(0, K, len(cuts))))
        bounds = cuts[1:] + [n[e]]
        for s0, s1, b in zip(cuts, bounds, sb[-1]):
            for i in range(s0, min(s1, n[e])):
                want[task[e, i], b, flags[e, i] & 0x3F] += 1
    tb = TraceBatch.from_arrays(np.sort(rng.uniform(0, 1e6, (E, ld)), axis=1), task, ss, sr,
                                n_events=n, seg_bucket=sb)
    got = selection_counts(tb, torch.as_tensor(flags, device=cuda), T, M, K).cpu().numpy()
    assert np.array_equal(got, want)
