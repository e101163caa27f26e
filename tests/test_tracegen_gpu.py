"""On-device workload generators (be_trace_gen / be_trace_gen_stable) vs the
statistical contract of the reference generators (pkg/tests/test_workload.py:
26-124 — the same checks, thresholds and sample sizes, applied per env).
numpy's PCG64 + ziggurat stream cannot be reproduced by Philox, so parity here
is distributional; the device traces replay bit-exactly through
the oracle like any other trace (test_rollout_gpu.py)."""
import math

import numpy as np
import pytest
import torch

from paper_2401_07886_b200 import CapacityError, InvalidParameterError, TraceBatch
from paper_2401_07886_b200.evalkit import scenario_names, scenario_suite

pytestmark = pytest.mark.gpu


def rows(tb):
    E = tb.n_envs
    n = tb.n_events.cpu().numpy() if tb.n_events is not None else np.full(E, tb.ld)
    arr = tb.arrival.cpu().numpy()
    tsk = tb.task.cpu().numpy()
    offs = tb.seg_offsets.cpu().numpy()
    ss = tb.seg_start.cpu().numpy()
    sr = tb.seg_rate.cpu().numpy()
    return [(arr[e, :n[e]], tsk[e, :n[e]], ss[offs[e]:offs[e + 1]], sr[offs[e]:offs[e + 1]])
            for e in range(E)]


def ks_exp(gaps, rate):
    g = np.sort(gaps)
    n = len(g)
    cdf = 1.0 - np.exp(-g * (rate / 1000.0))
    return max((np.arange(1, n + 1) / n - cdf).max(), (cdf - np.arange(0, n) / n).max())


def test_stable_per_segment_rate_and_tasks(cuda):
    # test_workload.py:27-32, :39-46
    tb = TraceBatch.generate("stable", 8, 4, seed=1, rates=[0.5, 2.0, 8.0], hold_seconds=200.0)
    for arr, tsk, ss, sr in rows(tb):
        assert list(sr) == [0.5, 2.0, 8.0]
        ends = list(ss[1:]) + [len(arr)]
        for k, rate in enumerate(sr):
            assert ends[k] - ss[k] == pytest.approx(rate * 200.0, rel=0.25)
            seg = arr[ss[k]:ends[k]]
            assert np.all((seg >= k * 200_000.0) & (seg < (k + 1) * 200_000.0))
        assert np.all(np.diff(arr) >= 0)
        assert set(tsk.tolist()) == {0, 1, 2, 3}
    sub = TraceBatch.generate("stable", 4, 4, seed=3, rates=[10.0], hold_seconds=100.0, task_ids=[2])
    assert all(set(r[1].tolist()) == {2} for r in rows(sub))


def test_stable_mean_gap_and_ks(cuda):
    # test_workload.py:34-37 (mean gap within 2%) and :60-74 (KS at the 1% level)
    tb = TraceBatch.generate("stable", 16, 1, seed=7, rates=[4.0], hold_seconds=2700.0)
    fails = 0
    for arr, _, _, _ in rows(tb):
        assert len(arr) > 10_001
        gaps = np.diff(arr[1:10_002])
        assert np.mean(gaps) == pytest.approx(250.0, rel=0.04)
        fails += ks_exp(gaps, 4.0) >= 1.628 / math.sqrt(len(gaps))
    assert fails <= 2  # 1% level over 16 independent envs


def test_stable_per_env_rates_and_truncation(cuda):
    rates = [[3.0 * (1 + k % 10)] for k in range(20)]
    tb = TraceBatch.generate("stable", 20, 4, seed=5, rates=rates, hold_seconds=4000.0,
                             ld=10_000, truncate=True)
    assert tb.n_events is None  # every env has >= 10k events in 4000 s at >= 3 req/s
    for e, (arr, _, ss, sr) in enumerate(rows(tb)):
        assert len(arr) == 10_000 and list(sr) == rates[e]
        assert np.mean(np.diff(arr)) == pytest.approx(1000.0 / rates[e][0], rel=0.06)
    with pytest.raises(CapacityError):
        TraceBatch.generate("stable", 2, 4, seed=5, rates=[30.0], hold_seconds=4000.0, ld=10_000)


def test_unpredictable_time_based(cuda):
    # test_workload.py:77-103: total count, bands 90/8/2 within 3 sigma, rates in range
    tb = TraceBatch.generate("unpredictable-time", 32, 4, seed=3, n_requests=10_000)
    assert tb.n_events is None and tb.ld == 10_000
    all_rates, lens, means = [], [], []
    for arr, tsk, ss, sr in rows(tb):
        assert len(arr) == 10_000 and ss[0] == 0 and np.all(np.diff(ss) > 0)
        assert np.all(np.diff(arr) >= 0) and arr[0] > 0
        assert np.all((sr >= 0.25) & (sr <= 48.0))
        all_rates.extend(sr.tolist())
        ends = np.append(ss[1:], len(arr))
        lens.extend((ends - ss)[:-1].tolist())
        means.extend((20.0 * sr[:-1]).tolist())
    r = np.array(all_rates)
    n = len(r)
    assert n >= 2_000
    for (lo, hi), p in zip(((0.25, 2.0), (2.0, 40.0), (40.0, 48.0)), (0.90, 0.08, 0.02)):
        cnt = int(np.sum((r >= lo) & ((r < hi) if hi < 48 else (r <= hi))))
        assert abs(cnt - n * p) < 3 * math.sqrt(n * p * (1 - p))
    # shifted geometric with mean 20 * rate: E[len / mean] = 1 (untruncated segments)
    ratio = np.array(lens) / np.array(means)
    assert np.mean(ratio) == pytest.approx(1.0, abs=4 * np.std(ratio) / math.sqrt(len(ratio)))


def test_unpredictable_request_based(cuda):
    # test_workload.py:106-124: geometric mean 500 within 5 %, rates in [1, 48]
    tb = TraceBatch.generate("unpredictable-request", 4, 4, seed=5, n_requests=600_000)
    for arr, _, ss, sr in rows(tb):
        assert len(arr) == 600_000
        assert np.all((sr >= 1.0) & (sr <= 48.0))
        lens = np.diff(np.append(ss, len(arr)))[:-1]  # drop the truncated final segment
        assert len(lens) >= 1_000
        assert np.mean(lens[:1_000]) == pytest.approx(500.0, rel=0.05)
    one = TraceBatch.generate("unpredictable-request", 2, 4, seed=2, n_requests=1)
    assert one.ld == 1 and int(one.seg_offsets[-1]) == 2


def test_same_global_env_same_trace(cuda):
    """Env k's trace depends only on (seed, global id): sharding-invariant (§8e)."""
    a = TraceBatch.generate("unpredictable-time", 16, 4, seed=9, n_requests=3000)
    b = TraceBatch.generate("unpredictable-time", 8, 4, seed=9, n_requests=3000, env_offset=8)
    ra, rb = rows(a), rows(b)
    for k in range(8):
        for x, y in zip(ra[8 + k], rb[k]):
            assert np.array_equal(x, y)
    c = TraceBatch.generate("unpredictable-time", 16, 4, seed=9, n_requests=3000)
    assert torch.equal(a.arrival, c.arrival) and torch.equal(a.task, c.task)


def test_scenarios_generate(cuda):
    for name in scenario_names():
        sc = scenario_suite(name)
        tb = TraceBatch.from_scenario(sc, 4, 4, seed=1)
        for arr, tsk, ss, sr in rows(tb):
            assert len(arr) > 0 and np.all(np.diff(arr) >= 0)
            if sc.task_ids is not None:
                assert set(tsk.tolist()) <= set(sc.task_ids)
            if sc.workload == "stable":
                assert list(sr) == list(sc.rates)


def test_rejects_bad_parameters(cuda):
    # test_workload.py:48-55 (InvalidParameterError), :201-209
    with pytest.raises(InvalidParameterError):
        TraceBatch.generate("stable", 1, 1, 0, rates=[], hold_seconds=10.0)
    with pytest.raises(InvalidParameterError):
        TraceBatch.generate("stable", 1, 1, 0, rates=[-1.0], hold_seconds=10.0)
    with pytest.raises(InvalidParameterError):
        TraceBatch.generate("stable", 1, 1, 0, rates=[1.0], hold_seconds=0.0)
    with pytest.raises(InvalidParameterError):
        TraceBatch.generate("unpredictable-time", 1, 4, 0, n_requests=0)
    with pytest.raises(InvalidParameterError):
        TraceBatch.generate("unpredictable-time", 1, 4, 0, task_ids=[4])
    with pytest.raises(ValueError):
        TraceBatch.generate("bursty", 1, 4, 0)
