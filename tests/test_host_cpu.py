"""Host-side logic that runs without a GPU: spec mirrors, validation errors,
BEQN1 checkpoints, config packing for the C ABI, sharding (gloo, world size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_07886_b200 import (CheckpointError, InvalidParameterError, ModelTierSpec, QNetwork,
                                   RewardSpec, StateEncoding, TaskSpec, default_tiers,
                                   load_checkpoint, make_cfg, save_checkpoint)
from paper_2401_07886_b200 import sharding, specs
from paper_2401_07886_b200.env import default_ring_capacity
from paper_2401_07886_b200.trainer import TrainConfig

import goldens


def test_tier_spec_validation_matches_reference():
    # simcore.py:31-37 / test_simcore.py:196-204
    for bad in [(0, 0, 1.0, 0.0, 1), (0, 1, 0.0, 0.0, 1), (0, 1, 1.0, -0.1, 1), (0, 1, 1.0, 0.0, 0)]:
        with pytest.raises(InvalidParameterError):
            ModelTierSpec(*bad)


def test_reward_spec_validation():
    with pytest.raises(ValueError):
        TaskSpec("x", 0.0)
    with pytest.raises(ValueError):
        RewardSpec(tasks=(TaskSpec("a", 40.0),), matrix=((1.5, 1.0),))
    assert RewardSpec.default().n_tasks == 4 and RewardSpec.default().n_tiers == 3


def test_default_tiers_are_the_shipped_calibration():
    t = default_tiers()
    assert [(x.alpha_ms, x.beta_ms, x.max_batch) for x in t] == [(4.75, 0.25, 128), (8.0, 1.2, 32),
                                                                 (28.0, 4.0, 8)]
    assert [x.max_batch for x in default_tiers(baseline=True)] == [160, 48, 12]


def test_checkpoint_roundtrip_and_errors(tmp_path):
    net = QNetwork.init_random(4, 3, 256, np.random.default_rng(0))
    p = str(tmp_path / "n.beqn")
    save_checkpoint(net, p)
    back = load_checkpoint(p)
    for a, b in zip(net.params(), back.params()):
        assert np.array_equal(a, b)
    raw = open(p, "rb").read()
    open(p, "wb").write(b"XXXX1\n" + raw.split(b"\n", 1)[1])
    with pytest.raises(CheckpointError):
        load_checkpoint(p)
    open(p, "wb").write(raw[:-8])
    with pytest.raises(CheckpointError, match="truncated"):
        load_checkpoint(p)
    open(p, "wb").write(raw + b"x")
    with pytest.raises(CheckpointError, match="trailing"):
        load_checkpoint(p)
    with pytest.raises(CheckpointError):
        load_checkpoint(str(tmp_path / "n2.beqn") if False else p, n_tasks=5)


def test_trained_fixture_loads():
    net = load_checkpoint(os.path.join(goldens.GOLDEN, "trained_seed7.beqn"))
    assert (net.n_tasks, net.n_tiers, net.hidden) == (4, 3, 256)
    ref = goldens.nets()["trained"]
    assert np.array_equal(net.w1, ref["w1"])


def test_make_cfg_packs_reference_objects():
    c = make_cfg(default_tiers(), RewardSpec.default(), StateEncoding(4, (128.0, 32.0, 8.0)),
                 estimator_mode="true-rate", ring_capacity=256)
    assert c.n_tiers == 3 and c.n_tasks == 4 and c.ring_capacity == 256
    assert c.tiers[2].alpha_ms == 28.0 and c.matrix[0 * 3 + 1] == 0.78
    assert c.estimator_true_rate == 1 and c.batch_scales[1] == 32.0
    with pytest.raises(InvalidParameterError):
        make_cfg(default_tiers(), RewardSpec.default(), estimator_mode="bogus")
    bad = [ModelTierSpec(1, 4, 4.75, 0.25, 128)]
    with pytest.raises(InvalidParameterError):
        make_cfg(bad, RewardSpec(tasks=(TaskSpec("a", 40.0),), matrix=((1.0,),)))


def test_ring_capacity_sizing():
    assert default_ring_capacity(10000, 4, 12, 1 << 40) == 16384
    cap = default_ring_capacity(10000, 65536, 12, 16 << 30)
    assert cap & (cap - 1) == 0 and 65536 * 12 * cap * 16 <= 16 << 30


def test_train_config_mirrors_reference():
    cfg = TrainConfig(total_iterations=1000)
    assert cfg.epsilon_at(0) == 1.0 and cfg.epsilon_at(250) == pytest.approx(0.05)
    with pytest.raises(ValueError):
        TrainConfig(batch_size=10, buffer_capacity=5)
    with pytest.raises(ValueError):
        TrainConfig(optimizer="rmsprop")


def test_event_rates_match_reference_rule():
    tr = specs.WorkloadTrace([specs.ArrivalEvent(float(i), 0) for i in range(6)],
                             [specs.SegmentMark(0, 1.0), specs.SegmentMark(2, 2.0),
                              specs.SegmentMark(2, 3.0), specs.SegmentMark(5, 4.0)], 0)
    assert tr.event_rates().tolist() == [1.0, 1.0, 3.0, 3.0, 3.0, 4.0]
    assert tr.segments() == [(0, 2, 1.0), (2, 5, 3.0), (5, 6, 4.0)]


def test_shard_range_partitions():
    for total, world in [(65536, 8), (10, 3), (5, 8)]:
        got = [sharding.shard_range(total, world, r) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_07886_b200.evalkit import ReduceResult
    E, K = 3, 2
    g = torch.Generator().manual_seed(rank)
    red = ReduceResult((1.0, 0.9), torch.randint(0, 100, (E, 2), generator=g),
                       torch.full((E,), 81, dtype=torch.int64),
                       torch.randint(0, 10, (E, K), generator=g),
                       torch.full((E, K), 50, dtype=torch.int64),
                       torch.rand((E, K), generator=g, dtype=torch.float64))
    tot = sharding.reduce_stats(red, torch.device("cpu"))
    mx = sharding.max_over_ranks(float(rank + 1), torch.device("cpu"))
    grad = torch.full((5,), float(rank + 1), dtype=torch.float64)
    sharding.allreduce_mean_(grad)
    params = torch.full((4,), float(rank), dtype=torch.float64)
    sharding.broadcast_params([params])
    out[rank] = (tot, mx, grad.tolist(), params.tolist(), red)
    dist.destroy_process_group()


def test_multiprocess_stats_reduce_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    (t0, m0, g0, p0, r0), (t1, m1, g1, p1, r1) = out[0], out[1]
    assert t0 == t1  # every rank holds identical totals
    assert m0 == m1 == 2.0
    assert g0 == g1 == [1.5] * 5
    assert p0 == p1 == [0.0] * 4
    wc = (r0.win_counts.sum(0) + r1.win_counts.sum(0)).tolist()
    assert t0["win_counts"] == wc and t0["n_windows"] == 6 * 81
    req = (r0.bucket_req.sum(0) + r1.bucket_req.sum(0)).numpy()
    miss = (r0.bucket_miss.sum(0) + r1.bucket_miss.sum(0)).numpy()
    assert t0["requests"] == req.tolist()
    assert t0["availability"] == pytest.approx((1 - miss / req).tolist())
    rws = r0.bucket_reward.sum(0).numpy() + r1.bucket_reward.sum(0).numpy()
    assert t0["mean_reward"] == pytest.approx((rws / req).tolist(), rel=1e-15)
