"""Evaluation reducer (be_reduce_eval) vs the oracle restatement of
evalkit.windowed / threshold_counts (evalkit.py:217-241) and the per-rate
miss fractions (evalkit.py:61-68): counts bit-exact, reward sums to 1e-12."""
import numpy as np
import pytest
import torch

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
                                         (64, 4096, False), (33, 25, True)])
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
