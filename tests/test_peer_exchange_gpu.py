"""Data-parallel learner with the peer-memory gradient exchange (be_train_iteration
phase 4, learner_xupdate_kernel) against the NCCL-style path (phase 3 + 1 +
host all-reduce of the gradients and the readiness gate + phase 2), emulated
in one process: two ranks on one GPU, each with its own learner, env batch and
CUDA stream, peers given as in-process device pointers.  Every rank must end
bit-identical to every other and to the all-reduce path."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2401_07886_b200 import RewardSpec, StateEncoding, default_tiers, _lib
from paper_2401_07886_b200.env import EnvBatch
from paper_2401_07886_b200.specs import QNetwork
from paper_2401_07886_b200.trainer import DeviceLearner, TrainConfig

pytestmark = pytest.mark.gpu


def make_rank(cfg, E, net, dev, r):
    tiers, rw = default_tiers(), RewardSpec.default()
    enc = StateEncoding(4, tuple(float(t.max_batch) for t in tiers))
    L = DeviceLearner(4, 3, cfg, E, 512, dev)
    L.set_params(net)
    env = EnvBatch(tiers, rw, E, enc, estimator_mode=cfg.estimator_mode, prior_rate=cfg.prior_rate,
                   ring_capacity=256, device=dev)
    tic = _lib.BeTrainIterCfg()
    tic.workload_seed, tic.policy_seed, tic.sample_seed = 11 + 100 * r, 12 + 100 * r, 13 + 100 * r
    tic.epsilon_start, tic.epsilon_end = cfg.epsilon_start, cfg.epsilon_end
    tic.epsilon_decay_steps = int(cfg.epsilon_decay_fraction * cfg.total_iterations)
    tic.updates_per_step = 2
    return L, env, tic


def run(L, env, tic, phase, uidx=0, use_gate=0):
    tic.phase, tic.update_index, tic.use_gate = phase, uidx, use_gate
    _lib.check(L._L.be_train_iteration(L.handle, env.handle, ctypes.byref(tic), _lib.stream_ptr()))


def test_peer_exchange_matches_allreduce_path(cuda):
    W, E, its = 2, 48, 220
    cfg = TrainConfig(batch_size=64, buffer_capacity=20_000, warmup=900, total_iterations=its, seed=5,
                      target_sync_every=7)
    net = QNetwork.init_random(4, 3, 256, np.random.default_rng(3))
    peer = [make_rank(cfg, E, net, cuda, r) for r in range(W)]
    ref = [make_rank(cfg, E, net, cuda, r) for r in range(W)]
    xm = [L.exchange_buffer() for L, _, _ in peer]
    for r, (L, _, _) in enumerate(peer):
        L.set_peers(r, xm)
    streams = [torch.cuda.Stream(cuda) for _ in range(W)]
    torch.cuda.synchronize()
    for _ in range(its):
        for r, (L, env, tic) in enumerate(peer):  # ranks run concurrently on their streams
            with torch.cuda.stream(streams[r]):
                run(L, env, tic, 4)
    # the all-reduce path, one rank after the other on the default stream
    min_size = max(cfg.batch_size, cfg.warmup)
    for _ in range(its):
        for L, env, tic in ref:
            run(L, env, tic, 3)
        for u in range(2):
            ready = min(int(L.ring_state[1] >= min_size) for L, _, _ in ref)
            for L, _, _ in ref:
                L.gate.fill_(ready)
            for L, env, tic in ref:
                run(L, env, tic, 1, u, 1)
            g = ref[0][0].grad + ref[1][0].grad  # all-reduce (sum), rank order
            for L, env, tic in ref:
                L.grad.copy_(g).mul_(1.0 / W)
                run(L, env, tic, 2, u, 1)
    torch.cuda.synchronize()
    for L, _, _ in peer + ref:
        L.check()
    p0 = peer[0][0].params.cpu()
    assert int(peer[0][0].counters[1]) > 100, "updates must have happened"
    for L, _, _ in peer[1:] + ref:
        assert torch.equal(L.params.cpu(), p0)
        assert torch.equal(L.target.cpu(), peer[0][0].target.cpu())
        assert L.counters[:4].tolist() == peer[0][0].counters[:4].tolist()
    for r in range(W):  # per-rank replay contents identical between the two paths
        assert torch.equal(peer[r][0].ring_rewards.cpu(), ref[r][0].ring_rewards.cpu())
        assert float(peer[r][0].loss[1]) == float(ref[r][0].loss[1])


def test_missing_peer_times_out_loudly(cuda):
    """A rank whose peer never publishes fails with an error after the bounded
    wait (2 s) instead of hanging the GPU; no update is applied."""
    cfg = TrainConfig(batch_size=64, buffer_capacity=20_000, warmup=64, total_iterations=4, seed=5)
    net = QNetwork.init_random(4, 3, 256, np.random.default_rng(3))
    (A, envA, ticA), (B, _, _) = [make_rank(cfg, 32, net, cuda, r) for r in range(2)]
    A.set_peers(0, [A.exchange_buffer(), B.exchange_buffer()])  # B never runs
    before = A.params.cpu().clone()
    run(A, envA, ticA, 4)
    with pytest.raises(_lib.CudaError, match="peer gradient exchange"):
        A.check()
    assert torch.equal(A.params.cpu(), before)
