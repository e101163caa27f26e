"""End-to-end StreamingEvaluator (pinned host traces -> copy stream -> fused
rollout + reducer -> pinned statistics) against the device-resident path."""
import os

import pytest
import torch

import goldens
from paper_2401_07886_b200 import (GreedyRollout, RewardSpec, StateEncoding, TraceBatch,
                                   default_tiers, load_checkpoint, reduce_eval)
from paper_2401_07886_b200.evalkit import StreamingEvaluator, pin_trace

pytestmark = pytest.mark.gpu


def test_streaming_matches_device_path(cuda):
    E, N, K = 512, 2000, 10
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    net = load_checkpoint(os.path.join(goldens.GOLDEN, "trained_seed7.beqn"))
    batches = []
    for seed in (3, 4, 5):
        rates = [3.0 * (1 + (e % K)) for e in range(E)]
        batches.append(TraceBatch.generate_stable(rates, N, 4, seed, device=cuda,
                                                  buckets=[e % K for e in range(E)]))
    ro = GreedyRollout(tiers, rw, E, N, enc, estimator_mode="true-rate", want_realized=False)
    want = []
    for tb in batches:
        o = ro.run(tb, net)
        want.append(reduce_eval(tb, o.flags, o.reward, n_buckets=K).totals())
    se = StreamingEvaluator(net, tiers, rw, E, N, enc, estimator_mode="true-rate", n_buckets=K,
                            ring_capacity=ro.ring_capacity, device=cuda)
    hosts = [pin_trace(tb) for tb in batches]
    for rnd in range(3):  # several outstanding submits, buffers and stat slots recycled
        handles = [se.submit(h) for h in hosts]
        got = [se.result(h).totals() for h in handles]
        for g, w in zip(got, want):
            assert g.keys() == w.keys()
            for k in w:
                assert str(g[k]) == str(w[k]), (rnd, k)
    assert se.h2d_bytes > E * N * 9 and se.d2h_bytes > 0


def test_streamed_rows_that_never_arrive_fail_loudly(cuda):
    """A chunk flag that is never written makes the rollout report an error after
    the bounded wait (5 s) instead of hanging or reading garbage silently."""
    from paper_2401_07886_b200 import CudaError
    E, N = 64, 500
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    net = load_checkpoint(os.path.join(goldens.GOLDEN, "trained_seed7.beqn"))
    tb = TraceBatch.generate_stable([3.0] * E, N, 4, 1, device=cuda)
    ro = GreedyRollout(tiers, rw, E, N, enc, estimator_mode="true-rate", want_realized=False,
                       ring_capacity=4096)
    flags = torch.zeros(4, dtype=torch.int32, device=cuda)
    flags[:2] = 7  # chunks 0-1 ready, 2-3 never
    ro.launch(tb, net, ready=(flags, 16, 7))
    with pytest.raises(CudaError, match="never became ready"):
        ro.env.check()


def test_streaming_overflow_raises_at_result(cuda):
    """A ring overflow inside a pipelined batch surfaces at that batch's result()
    (the device status travels with the statistics; no stream-wide sync per batch)."""
    from paper_2401_07886_b200 import CapacityError
    E, N = 64, 3000
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    tb = TraceBatch.generate_stable([30.0] * E, N, 4, 2, device=cuda)  # 10x load: queues grow
    se = StreamingEvaluator(2, tiers, rw, E, N, enc, estimator_mode="true-rate", ring_capacity=8,
                            device=cuda)  # static large tier floods its 4 replicas
    h = se.submit(pin_trace(tb))
    with pytest.raises(CapacityError):
        se.result(h)
