"""Multi-rank paths on one GPU (the GPU box has one device; NCCL refuses two
ranks on one GPU, so these use the gloo backend with CUDA tensors — the
collectives are the same torch.distributed calls the NCCL path makes):
  * data-parallel learner (run_training(world=...)): gradients all-reduced
    between backward and Adam -> replicas stay bit-identical, shards differ;
  * the same learner with exchange="peer" (gradients read from the peers'
    exchange buffers through CUDA IPC, no collective per update);
  * bench.py under torchrun with 2 ranks: env-sharded rollout, max-over-ranks
    timing, end-of-run statistics all-reduce, one JSON line from rank 0."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dp_worker(rank, world, port, out, exchange="nccl"):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_07886_b200 import RewardSpec, default_tiers
    from paper_2401_07886_b200.trainer import TrainConfig, run_training
    cfg = TrainConfig(batch_size=64, buffer_capacity=20_000, warmup=500, total_iterations=120,
                      log_every=60, seed=4)
    res = run_training(default_tiers(), RewardSpec.default(), cfg, n_envs=16, updates_per_step=1,
                       world=dist.group.WORLD, exchange=exchange)
    out[rank] = ([p.copy() for p in res.net.params()], res.updates, res.transitions,
                 [(r.loss, r.mean_recent_reward) for r in res.log])
    dist.destroy_process_group()


def test_data_parallel_learner_replicas_identical(cuda):
    world, port = 2, _port()
    out = mp.Manager().dict()
    mp.spawn(_dp_worker, args=(world, port, out), nprocs=world, join=True)
    (p0, u0, t0, l0), (p1, u1, t1, l1) = out[0], out[1]
    assert u0 == u1 > 0
    for a, b in zip(p0, p1):  # one all-reduced gradient per update: identical replicas
        assert np.array_equal(a, b)
    assert len(l0) == len(l1) == 2
    assert t0 != t1 or l0 != l1  # the env shards (and their batches) are independent


def test_peer_exchange_two_processes_matches_allreduce(cuda):
    """exchange="peer": the ranks swap CUDA IPC handles of their exchange buffers
    once and every update reads the peers' gradients from their memory (two
    processes on one GPU here; NVLink peer memory across GPUs).  Same replicas,
    bit for bit, as the all-reduce path on the same seeds."""
    world = 2
    res = {}
    for exchange in ("nccl", "peer"):
        out = mp.Manager().dict()
        mp.spawn(_dp_worker, args=(world, _port(), out, exchange), nprocs=world, join=True)
        res[exchange] = (out[0], out[1])
    (p0, u0, t0, l0), (p1, u1, t1, l1) = res["peer"]
    assert u0 == u1 > 0
    for a, b in zip(p0, p1):
        assert np.array_equal(a, b)
    for r in range(world):
        pa, ua, ta, la = res["peer"][r]
        pb, ub, tb, lb = res["nccl"][r]
        assert (ua, ta, la) == (ub, tb, lb)
        for a, b in zip(pa, pb):
            assert np.array_equal(a, b)


def _bench(args, world, env=None):
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}"]
    else:
        cmd = [sys.executable]
    cmd += [os.path.join(ROOT, "bench.py"), "--gpus", str(world)] + args
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    return json.loads(lines[0])


def test_bench_two_ranks_one_gpu(cuda, tmp_path):
    """Config 4's split: the same 4,096 global envs on one rank and sharded over two
    (by global id, traces keyed by global id): the all-reduced integer statistics
    are bit-equal, rewards equal up to the rank-order summation; both runs pass the
    in-line oracle parity check."""
    env = dict(os.environ, BE_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    args = ["--steps", "2", "--warmup", "3", "--envs", "4096", "--requests", "2000",
            "--no-cpu-baseline", "--no-training", "--parity-envs", "8"]
    d1 = _bench(args, 1, env)
    d2 = _bench(args, 2, env)
    for d, n in ((d1, 1), (d2, 2)):
        assert d["n_gpus"] == n and d["config"]["total_envs"] == 4096 and d["scaling"] == "strong"
        assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["stats_identical_to_resident_run"]
        assert d["parity"]["mismatches"] == 0 and d["parity"]["envs"] >= 8
    assert d2["config"]["envs_per_gpu"] == 2048
    assert d2["weak_scaling"]["envs_per_gpu"] == 4096 and d2["weak_scaling"]["value"] > 0
    r1, r2 = d1["results"], d2["results"]
    assert sum(r2["requests"]) == 4096 * 2000
    for k in ("win_counts", "n_windows", "requests", "misses"):
        assert r1[k] == r2[k], k
    np.testing.assert_allclose(r1["mean_reward"], r2["mean_reward"], rtol=1e-12)
