"""DQN training on the GPU (drop-in for besteffort.trainer).

  TrainConfig                 trainer.py:39-90 (same fields, validation, epsilon_at)
  run_training                trainer.py:333-406 — E environments step in lockstep; each
                              vectorised iteration routes one request per env (epsilon-
                              greedy), commits resolved transitions into the device
                              replay ring and takes `updates_per_step` learner updates
  DeviceLearner               ReplayBuffer + _StepKernel + Adam/SGD + target sync on the
                              device (be_learner_*), fp64, deterministic per batch
  train_step_batch            one update on an explicit batch (parity with the reference)

Update-to-data ratio: the reference takes one update per routed request (one env). With
E envs per iteration this module takes `updates_per_step` updates per E requests (UTD =
updates_per_step / E); with n_envs=1 it is exactly the reference's schedule.
Randomness (arrivals, epsilon, sampling, init) uses Philox, so runs are reproducible
but not bit-identical to numpy PCG64 streams (statistical parity).
"""
from __future__ import annotations

import ctypes
import math
from collections import deque
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .env import EnvBatch, StepRecords
from .specs import QNetwork, StateEncoding


@dataclass
class TrainConfig:
    discount: float = 0.99
    learning_rate: float = 1e-4
    batch_size: int = 1024
    target_sync_every: int = 500
    total_iterations: int = 200_000
    epsilon_start: float = 1.0
    epsilon_end: float = 0.05
    epsilon_decay_fraction: float = 0.25
    buffer_capacity: int = 500_000
    warmup: int = 10_000
    optimizer: str = "adam"
    loss: str = "huber"
    hidden: int = 256
    seed: int = 0
    log_every: int = 10_000
    rate_low: float = 0.25
    rate_high: float = 48.0
    regime_cadence: str = "equal-time"
    regime_mean_seconds: float = 20.0
    regime_mean_requests: float = 100.0
    estimator_mode: str = "true-rate"
    prior_rate: float = 1.0

    def __post_init__(self):  # trainer.py:74-83
        if not 0.0 < self.discount < 1.0:
            raise ValueError("discount must lie in (0, 1)")
        if self.batch_size > self.buffer_capacity:
            raise ValueError("batch_size must not exceed buffer capacity")
        if self.batch_size < 1 or self.total_iterations < 0:
            raise ValueError("batch_size must be >= 1 and total_iterations >= 0")
        if not 0.0 <= self.epsilon_end <= self.epsilon_start <= 1.0:
            raise ValueError("need 0 <= epsilon_end <= epsilon_start <= 1")
        if self.rate_low <= 0 or self.rate_high < self.rate_low:
            raise ValueError("need 0 < rate_low <= rate_high")
        if self.optimizer not in ("adam", "sgd"):
            raise ValueError("optimizer must be 'adam' or 'sgd'")
        if self.regime_cadence not in ("equal-time", "requests"):
            raise ValueError("regime_cadence must be 'equal-time' or 'requests'")

    def epsilon_at(self, iteration: int) -> float:  # trainer.py:85-90
        decay_steps = int(self.epsilon_decay_fraction * self.total_iterations)
        if decay_steps <= 0:
            return self.epsilon_end
        frac = min(1.0, iteration / decay_steps)
        return self.epsilon_start + (self.epsilon_end - self.epsilon_start) * frac


@dataclass
class LogRow:
    step: int
    loss: float
    mean_recent_reward: float
    epsilon: float


@dataclass
class TrainResult:
    net: QNetwork
    log: list = field(default_factory=list)
    updates: int = 0
    transitions: int = 0
    max_inflight: int = 0  # most decisions any request stayed unresolved (pending store high-water)


class DeviceLearner:
    """be_learner handle: online/target nets, Adam state, replay ring, pending store."""

    def __init__(self, n_tasks: int, n_tiers: int, cfg: TrainConfig, n_envs: int = 1,
                 pending_capacity: int = 4096, device=None):
        self.device = _lib.require_cuda(device)
        self.cfg = cfg
        self.n_tasks, self.n_tiers, self.n_envs = n_tasks, n_tiers, int(n_envs)
        self.D = n_tasks + n_tiers + 1
        self.P = int(pending_capacity)
        c = _lib.BeLearnerCfg()
        c.n_tasks, c.n_tiers, c.hidden, c.n_envs = n_tasks, n_tiers, cfg.hidden, self.n_envs
        c.replay_capacity = int(cfg.buffer_capacity)
        c.pending_capacity = self.P
        c.batch = int(cfg.batch_size)
        c.warmup = int(cfg.warmup)
        c.target_sync_every = int(cfg.target_sync_every)
        c.discount, c.learning_rate = float(cfg.discount), float(cfg.learning_rate)
        c.adam = 1 if cfg.optimizer == "adam" else 0
        c.huber = 1 if cfg.loss == "huber" else 0
        c.rate_low, c.rate_high = float(cfg.rate_low), float(cfg.rate_high)
        c.regime_equal_time = 1 if cfg.regime_cadence == "equal-time" else 0
        c.regime_mean_seconds = float(cfg.regime_mean_seconds)
        c.regime_mean_requests = float(cfg.regime_mean_requests)
        self._L = _lib.load()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.be_learner_create(ctypes.byref(c), self.device.index or 0,
                                                 ctypes.byref(h)))
        self._h = h
        self.views = _lib.BeLearnerViews()
        _lib.check(self._L.be_learner_views(self._h, ctypes.byref(self.views)))
        v = self.views
        self.nparam = v.nparam
        self.params = _wrap(v.params, (self.nparam,), torch.float64, self.device)
        self.grad = _wrap(v.grad, (self.nparam,), torch.float64, self.device)
        self.target = _wrap(v.target.w1, (self.nparam,), torch.float64, self.device)
        self.gate = _wrap(v.gate, (1,), torch.int64, self.device)
        self.loss = _wrap(v.loss, (2,), torch.float64, self.device)
        self.counters = _wrap(v.counters, (8,), torch.int64, self.device)
        self.ring_state = _wrap(v.ring_state, (8,), torch.int64, self.device)
        C = int(cfg.buffer_capacity)
        self.ring_rewards = _wrap(v.ring_rewards, (C,), torch.float64, self.device)
        self.ring_states = _wrap(v.ring_states, (C, self.D), torch.float64, self.device)
        self.ring_next_states = _wrap(v.ring_next_states, (C, self.D), torch.float64, self.device)
        self.ring_actions = _wrap(v.ring_actions, (C,), torch.uint8, self.device)
        self.ring_cont = _wrap(v.ring_cont, (C,), torch.float64, self.device)
        self.workload_state = _wrap(v.workload_state, (self.n_envs, 3), torch.float64, self.device)
        self.pending_x = _wrap(v.pending_x, (self.P, self.n_envs, self.D), torch.float64, self.device)
        self.pending_action = _wrap(v.pending_action, (self.P, self.n_envs), torch.uint8, self.device)
        self.pending_flags = _wrap(v.pending_flags, (self.n_envs, self.P), torch.uint8, self.device)
        self.pending_reward = _wrap(v.pending_reward, (self.n_envs, self.P), torch.float64, self.device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.be_learner_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ parameters
    def set_params(self, net) -> None:
        net = QNetwork.from_any(net)
        arrs = [np.ascontiguousarray(a, np.float64) for a in (net.w1, net.b1, net.w2, net.b2)]
        ts = [torch.from_numpy(a).to(self.device) for a in arrs]
        _lib.check(self._L.be_learner_set_params(self._h, *(t.data_ptr() for t in ts),
                                                 _lib.stream_ptr()))
        torch.cuda.current_stream().synchronize()

    @property
    def handle(self):
        return self._h

    def online_weights(self) -> _lib.BeQWeights:
        return self.views.online

    def net(self) -> QNetwork:
        p = self.params.cpu().numpy()
        D, H, M = self.D, self.cfg.hidden, self.n_tiers
        o = 0
        w1 = p[o:o + D * H].reshape(D, H); o += D * H
        b1 = p[o:o + H]; o += H
        w2 = p[o:o + H * M].reshape(H, M); o += H * M
        b2 = p[o:o + M]
        return QNetwork(self.n_tasks, M, w1.copy(), b1.copy(), w2.copy(), b2.copy())

    def target_net(self) -> QNetwork:
        v = self.views.target
        D, H, M = self.D, self.cfg.hidden, self.n_tiers
        w = [_wrap(ptr, shape, torch.float64, self.device).cpu().numpy().copy()
             for ptr, shape in ((v.w1, (D, H)), (v.b1, (H,)), (v.w2, (H, M)), (v.b2, (M,)))]
        return QNetwork(self.n_tasks, M, *w)

    # ------------------------------------------------------------ steps
    def backward(self, seed: int, counter: int, sample_idx: Optional[torch.Tensor] = None):
        _lib.check(self._L.be_learner_backward(self._h, seed & (2**64 - 1), counter & (2**64 - 1),
                                               _lib.ptr(sample_idx), _lib.stream_ptr()))

    def backward_batch(self, states, actions, rewards, next_states, cont):
        dev = self.device
        t = [torch.as_tensor(np.ascontiguousarray(x, dt), device=dev) for x, dt in
             ((states, np.float64), (actions, np.uint8), (rewards, np.float64),
              (next_states, np.float64), (cont, np.float64))]
        _lib.check(self._L.be_learner_backward_batch(self._h, *(x.data_ptr() for x in t),
                                                     int(t[0].shape[0]), _lib.stream_ptr()))
        self._keep = t

    def apply(self, explicit_batch: bool = False) -> None:
        _lib.check(self._L.be_learner_apply(self._h, 1 if explicit_batch else 0, _lib.stream_ptr()))

    def commit(self, step: int) -> None:
        _lib.check(self._L.be_learner_commit(self._h, int(step), _lib.stream_ptr()))

    def workload(self, seed: int, step: int, arrival, task, rate) -> None:
        _lib.check(self._L.be_learner_workload(self._h, seed & (2**64 - 1), int(step),
                                               arrival.data_ptr(), task.data_ptr(), rate.data_ptr(),
                                               _lib.stream_ptr()))

    def check(self) -> None:
        _lib.check(self._L.be_learner_check(self._h, _lib.stream_ptr()))

    # ------------------------------------------------------------ peer exchange (DP)
    def exchange_buffer(self) -> int:
        p = ctypes.c_void_p()
        _lib.check(self._L.be_learner_exchange_buffer(self._h, ctypes.byref(p), None))
        return int(p.value)

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _lib.check(self._L.be_learner_ipc_handle(self._h, buf))
        return buf.raw

    def set_peers(self, rank: int, xmems) -> None:
        """In-process peers: every rank's exchange_buffer() (xmems[rank] = own)."""
        arr = (ctypes.c_uint64 * len(xmems))(*[int(x) for x in xmems])
        _lib.check(self._L.be_learner_set_peers(self._h, len(xmems), int(rank), arr))

    def open_peers_ipc(self, rank: int, handles) -> None:
        """Peers in other processes: every rank's ipc_handle(), in rank order."""
        blob = b"".join(handles)
        _lib.check(self._L.be_learner_open_peers_ipc(self._h, len(handles), int(rank), blob))

    @property
    def size(self) -> int:
        return int(self.ring_state[1])


def _wrap(ptr: int, shape, dtype, device) -> torch.Tensor:
    """Zero-copy torch view of device memory owned by the C library."""
    n = int(np.prod(shape))
    esz = torch.empty((), dtype=dtype).element_size()
    t = torch.as_tensor(_DevPtr(ptr, n * esz, device), device=device)
    return t.view(dtype).view(*shape)


class _DevPtr:
    """__cuda_array_interface__ exporter for a raw device allocation (bytes)."""

    def __init__(self, ptr: int, nbytes: int, device):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def run_training(tiers, reward_spec, cfg: TrainConfig, encoding=None, init_net=None,
                 completion_log=None, *, n_envs: int = 1, updates_per_step: int = 1,
                 pending_capacity: Optional[int] = None, ring_capacity: int = 1024, device=None,
                 world=None, mode: str = "device", graph_chunk: int = 0,
                 timing: Optional[dict] = None, exchange: str = "nccl",
                 router: str = "fp64") -> TrainResult:
    """trainer.py:333-406 on the GPU for `n_envs` lockstep environments.

    Every iteration: TrainingWorkload arrivals (Philox), one env step with
    epsilon-greedy routing, deferred-reward commits into the replay ring, and
    `updates_per_step` learner updates (batch `cfg.batch_size`).
    mode:
      "device" (default) be_train_iteration — every per-iteration value lives on
               the device and each update is one fused kernel; launched eagerly;
      "graph"  the same iterations captured once (`graph_chunk` at a time) in a
               CUDA graph and replayed (B200, E = 4096, batch 512: ~15k it/s vs
               ~14k eager — 6 dependent launches per iteration, ~47 us of kernels;
               launches use programmatic dependent launch, PDL);
      "host"   the step-by-step C ABI (workload / env step / commit / backward /
               apply) driven from Python — the reference loop's structure.
    All three give bit-identical results for the same seed.
    `world`: optional torch.distributed group — gradients are all-reduced (mean)
    between backward and the optimizer step (data-parallel learner; always runs
    as "device": readiness is all-reduced so every rank updates in the same
    iterations, and the collectives stay outside any graph).
    `exchange` (with `world`): "nccl" — gradients all-reduced by NCCL between the
    backward and the optimizer launches (readiness all-reduced too); "peer" — one
    update kernel per rank exchanges the gradients through the ranks' exchange
    buffers in peer memory (CUDA IPC handles swapped once over `world`), no
    collective on the update path, graph-capturable (be_train_iteration phase 4).
    `router`: "fp64" — the decision is made inside the env step (fp64 Q);
    "tc" — the step is split around the tensor-core router: observe + encode, then
    be_qnet_route_tc's certified tcgen05 forward (fp64 re-evaluation of the states it
    cannot certify) on the E states, then submit — the same decisions and exploration
    draws, so the same training run bit for bit (test); it pays off for large
    lockstep batches.
    `timing`: optional dict, receives the device time of the iteration loop
    ("loop_ms", CUDA events on the launching stream; setup and the one-time graph
    capture excluded, intermediate log rows included, the final one excluded)."""
    n_tasks, n_tiers = len(reward_spec.tasks), len(reward_spec.matrix[0])
    if len(tiers) != n_tiers:
        raise ValueError("tier count must match reward matrix width")
    if mode not in ("graph", "device", "host"):
        raise ValueError("mode must be 'graph', 'device' or 'host'")
    if completion_log is not None:
        # the audit trail is harvested per iteration from the pending store: the
        # host-driven loop (same results as the device / graph modes)
        if world is not None:
            raise ValueError("completion_log is not supported with a data-parallel world")
        mode = "host"
    if exchange not in ("nccl", "peer"):
        raise ValueError("exchange must be 'nccl' or 'peer'")
    if router not in ("fp64", "tc"):
        raise ValueError("router must be 'fp64' or 'tc'")
    if encoding is None:
        encoding = StateEncoding(n_tasks=n_tasks, batch_scales=tuple(float(t.max_batch) for t in tiers))
    dev = _lib.require_cuda(device)
    E = int(n_envs)
    if pending_capacity is None:
        pending_capacity = default_pending_capacity(E, n_tasks + n_tiers + 1)
    learner = DeviceLearner(n_tasks, n_tiers, cfg, E, pending_capacity, dev)
    if init_net is None:
        rng = np.random.default_rng(np.random.SeedSequence(cfg.seed).spawn(4)[0])
        init_net = QNetwork.init_random(n_tasks, n_tiers, cfg.hidden, rng)
    else:
        init_net = QNetwork.from_any(init_net)
        if init_net.n_tasks != n_tasks or init_net.n_tiers != n_tiers:
            raise ValueError("init_net dimensions do not match the environment")
    learner.set_params(init_net)
    if world is not None:
        import torch.distributed as dist
        dist.broadcast(learner.params, 0)
        dist.broadcast(learner.target, 0)
        if exchange == "peer":
            handles = [None] * dist.get_world_size()
            dist.all_gather_object(handles, learner.ipc_handle())
            learner.open_peers_ipc(dist.get_rank(), handles)
            torch.cuda.synchronize(dev)
            dist.barrier()
            if mode == "host":
                mode = "device"
        else:
            # the DP update gate (all ranks update in the same iterations) lives in the
            # device-resident iteration; the collective stays outside any graph
            mode = "device"
    env = EnvBatch(tiers, reward_spec, E, encoding, estimator_mode=cfg.estimator_mode,
                   prior_rate=cfg.prior_rate, ring_capacity=ring_capacity, device=dev)
    # SeedSequence(seed).spawn(4) -> init, env, policy, sample (trainer.py:351-353); a
    # data-parallel rank r > 0 owns a different env shard: its streams are spawned from
    # SeedSequence(seed, spawn_key=(r,)) so every rank draws independent arrivals
    rank = 0
    if world is not None:
        import torch.distributed as dist
        rank = dist.get_rank()
    root = np.random.SeedSequence(cfg.seed) if rank == 0 else np.random.SeedSequence(cfg.seed, spawn_key=(rank,))
    seeds = [int(s.generate_state(1, np.uint64)[0]) for s in root.spawn(4)]
    wl_seed, pol_seed, smp_seed = seeds[1], seeds[2], seeds[3]
    log = []
    total = int(cfg.total_iterations)
    log_every = max(1, int(cfg.log_every))

    def log_row(it):
        learner.check()
        env.check()
        size = learner.size
        k = min(size, 1000)
        cur = int(learner.ring_state[0])
        idx = (cur - 1 - torch.arange(k, device=learner.ring_rewards.device)) % cfg.buffer_capacity
        mean_recent = float(learner.ring_rewards[idx].mean()) if k else math.nan
        gs = int(learner.counters[1])
        loss = float(learner.loss[1]) if gs > 0 else math.nan
        log.append(LogRow(it + 1, loss, mean_recent, cfg.epsilon_at(it)))

    t_begin = torch.cuda.Event(enable_timing=True)
    t_begin.record()
    if mode == "host":
        _run_host_loop(learner, env, cfg, E, updates_per_step, world, wl_seed, pol_seed, smp_seed,
                       log_every, log_row, completion_log, router)
    else:
        tic = _lib.BeTrainIterCfg()
        tic.workload_seed, tic.policy_seed, tic.sample_seed = wl_seed, pol_seed, smp_seed
        tic.epsilon_start, tic.epsilon_end = float(cfg.epsilon_start), float(cfg.epsilon_end)
        tic.epsilon_decay_steps = int(cfg.epsilon_decay_fraction * total)
        tic.updates_per_step = int(updates_per_step)
        tic.router = 1 if router == "tc" else 0
        min_size = max(int(cfg.batch_size), int(cfg.warmup))
        gate_b = torch.empty(1, dtype=torch.bool, device=dev)

        def iteration():
            if world is not None and exchange == "peer":
                tic.phase, tic.update_index, tic.use_gate = 4, 0, 0
                _lib.check(learner._L.be_train_iteration(learner.handle, env.handle, ctypes.byref(tic),
                                                         _lib.stream_ptr()))
                return
            if world is None:
                tic.phase, tic.update_index = 0, 0
                _lib.check(learner._L.be_train_iteration(learner.handle, env.handle, ctypes.byref(tic),
                                                         _lib.stream_ptr()))
                return
            import torch.distributed as dist
            tic.phase, tic.update_index, tic.use_gate = 3, 0, 1
            _lib.check(learner._L.be_train_iteration(learner.handle, env.handle, ctypes.byref(tic),
                                                     _lib.stream_ptr()))
            for u in range(updates_per_step):
                # every rank updates in the same iterations: readiness all-reduced (MIN)
                torch.ge(learner.ring_state[1:2], min_size, out=gate_b)
                learner.gate.copy_(gate_b)
                dist.all_reduce(learner.gate, op=dist.ReduceOp.MIN)
                tic.phase, tic.update_index = 1, u
                _lib.check(learner._L.be_train_iteration(learner.handle, env.handle, ctypes.byref(tic),
                                                         _lib.stream_ptr()))
                dist.all_reduce(learner.grad)
                learner.grad.mul_(1.0 / dist.get_world_size())
                tic.phase = 2
                _lib.check(learner._L.be_train_iteration(learner.handle, env.handle, ctypes.byref(tic),
                                                         _lib.stream_ptr()))

        G = 1
        graph = None
        if mode == "graph":
            G = graph_chunk or max(d for d in range(1, 65) if log_every % d == 0)
            if G > 1 and total >= G:
                # capture (host-side, like compiling) before the timed loop starts: the
                # graph records G iterations, each replay runs them on the device
                graph = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(device=dev)
                side.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.graph(graph, stream=side):
                    for _ in range(G):
                        iteration()
                torch.cuda.current_stream(dev).wait_stream(side)
        t_begin = torch.cuda.Event(enable_timing=True)
        t_begin.record()
        it = 0
        while it < total:
            seg_end = min(total, (it // log_every + 1) * log_every)
            if graph is not None:
                while seg_end - it >= G:
                    graph.replay()
                    it += G
            while it < seg_end:
                iteration()
                it += 1
            if it == total:  # device work of the loop ends here (the last log row is host-side)
                t_end = torch.cuda.Event(enable_timing=True)
                t_end.record()
            if it % log_every == 0:
                log_row(it - 1)
    if total == 0 or mode == "host":
        t_end = torch.cuda.Event(enable_timing=True)
        t_end.record()
    learner.check()
    env.check()
    if timing is not None:
        timing["loop_ms"] = t_begin.elapsed_time(t_end)
    res = TrainResult(net=learner.net(), log=log, updates=int(learner.counters[1]),
                      transitions=int(learner.ring_state[2]), max_inflight=int(learner.ring_state[4]))
    learner.close()
    env.close()
    return res


def default_pending_capacity(n_envs: int, input_dim: int, budget_bytes: float = 8e9) -> int:
    """Decisions a request may stay unresolved (the pending store is [P][E] states +
    actions + rewards + flags): the largest power of two in [4096, 65536] within
    `budget_bytes`.  Exploration can overload a tier for long stretches — the
    config-3 recipe (4096 envs, 200k iterations) peaked at 6,430 decisions
    (profiles/r2_config3_policies.json); the reference's dict has no bound."""
    per = float(n_envs) * (8 * input_dim + 1 + 1 + 8)
    p = 65536
    while p > 4096 and p * per > budget_bytes:
        p //= 2
    return p


def _run_host_loop(learner, env, cfg, E, updates_per_step, world, wl_seed, pol_seed, smp_seed,
                   log_every, log_row, completion_log=None, router="fp64"):
    """The reference loop's structure (trainer.py:374-404), one C-ABI call per stage.

    completion_log (trainer.py:381-383): (request id, task, tier, realized ms/token,
    reward) of every completed request.  A request's pending slot (id mod P) is final
    once the slot is about to be reused (a request unresolved after P decisions is an
    error), so slot (it + 1) mod P is harvested after iteration it and the last P
    slots after the loop; entries are in request-id order (env-major within an id),
    not in the reference's completion-time order."""
    dev = learner.device
    P = learner.P
    rec = _PendingRecords(learner, want_realized=completion_log is not None)
    audit = _AuditHarvest(learner, rec, completion_log) if completion_log is not None else None
    arrival = torch.empty(E, dtype=torch.float64, device=dev)
    task = torch.empty(E, dtype=torch.uint8, device=dev)
    rate = torch.empty(E, dtype=torch.float64, device=dev)
    W = learner.online_weights()
    tc_ws = None
    if router == "tc":
        L = learner._L
        tc_ws = torch.empty((int(L.be_qnet_route_tc_workspace_bytes(cfg.hidden)) + 15) // 16 * 4,
                            dtype=torch.float32, device=dev)
    for it in range(cfg.total_iterations):
        learner.workload(wl_seed, it, arrival, task, rate)
        slot = it % P
        if router == "tc":
            _env_step_tc(env, learner, arrival, task, rate, W, cfg.epsilon_at(it), pol_seed, it, rec,
                         learner.pending_x[slot], learner.pending_action[slot], tc_ws)
        else:
            _env_step(env, arrival, task, rate, W, cfg.epsilon_at(it), pol_seed, it, rec,
                      learner.pending_x[slot], learner.pending_action[slot])
        learner.commit(it)
        for u in range(updates_per_step):
            learner.backward(smp_seed, it * updates_per_step + u)
            if world is not None:
                import torch.distributed as dist
                dist.all_reduce(learner.grad)
                learner.grad.mul_(1.0 / dist.get_world_size())
            learner.apply()
        learner.counters[3] += 1  # keep the device iteration index in step (views.counters[3])
        if audit is not None:
            audit.slot(it + 1 - P)
        if (it + 1) % log_every == 0:
            log_row(it)
    if audit is not None:
        for j in range(max(0, cfg.total_iterations - P + 1), cfg.total_iterations):
            audit.slot(j)
        audit.flush()


class _AuditHarvest:
    """Collects completion_log rows from the learner's pending store (device
    tensors staged per request id, copied to the host in blocks)."""

    def __init__(self, learner, rec, out):
        self.L, self.rec, self.out = learner, rec, out
        self.T = learner.n_tasks
        self.rows, self.ids = [], []

    def slot(self, j):
        if j < 0:
            return
        s = j % self.L.P
        f = self.rec.flags[:, s]
        done = (f & 0x60) != 0  # completed (0x40) or already committed (0x20)
        task = self.L.pending_x[s, :, :self.T].argmax(dim=1)
        self.rows.append(torch.stack([done.double(), task.double(),
                                      self.L.pending_action[s].double(),
                                      self.rec.realized[:, s], self.rec.reward[:, s]]))
        self.ids.append(j)
        if len(self.rows) >= 4096:
            self.flush()

    def flush(self):
        if not self.rows:
            return
        blk = torch.stack(self.rows).cpu().numpy()  # [n ids][5][E]
        for j, r in zip(self.ids, blk):
            for e in np.nonzero(r[0])[0]:
                self.out.append((j, int(r[1, e]), int(r[2, e]), float(r[3, e]), float(r[4, e])))
        self.rows, self.ids = [], []


class _PendingRecords:
    """StepRecords view onto the learner's pending reward/flag store (rec_ld = P)."""

    def __init__(self, learner: DeviceLearner, want_realized: bool = False):
        self.ld = learner.P
        self.flags = learner.pending_flags
        self.reward = learner.pending_reward
        self.realized = (torch.full_like(learner.pending_reward, float("nan"))
                         if want_realized else None)

    def struct(self) -> _lib.BeRecords:
        r = _lib.BeRecords()
        r.flags = self.flags.data_ptr()
        r.reward = self.reward.data_ptr()
        r.realized = _lib.ptr(self.realized)
        return r


def _env_step(env: EnvBatch, arrival, task, rate, W, epsilon, seed, counter, rec, x_out, a_out):
    E, M = env.n_envs, env.n_tiers
    r = rec.struct()
    _lib.check(env._L.be_env_step(env.handle, arrival.data_ptr(), task.data_ptr(), rate.data_ptr(),
                                  None, ctypes.byref(W), -1, float(epsilon), seed & (2**64 - 1),
                                  counter & (2**64 - 1), rec.ld, ctypes.byref(r), None, None,
                                  a_out.data_ptr(), None, x_out.data_ptr(), _lib.stream_ptr()))


def _env_step_tc(env: EnvBatch, learner, arrival, task, rate, W, epsilon, seed, counter, rec, x_out, a_out,
                 workspace):
    """The split step of router="tc": observe + encode into the pending slot, the
    tensor-core router on it (same epsilon / Philox draws as the fused step), submit."""
    L = env._L
    r = rec.struct()
    _lib.check(L.be_env_step_observe(env.handle, arrival.data_ptr(), task.data_ptr(), rate.data_ptr(), rec.ld,
                                     ctypes.byref(r), x_out.data_ptr(), None, None, _lib.stream_ptr()))
    _lib.check(L.be_qnet_route_tc(ctypes.byref(W), learner.n_tasks, learner.n_tiers, x_out.data_ptr(),
                                  env.n_envs, float(epsilon), seed & (2**64 - 1), counter & (2**64 - 1), None,
                                  a_out.data_ptr(), workspace.data_ptr(), None, _lib.stream_ptr()))
    _lib.check(L.be_env_step_submit(env.handle, arrival.data_ptr(), task.data_ptr(), a_out.data_ptr(), rec.ld,
                                    ctypes.byref(r), _lib.stream_ptr()))


def fine_tune(net, reward_spec, cfg: TrainConfig, tiers, encoding=None, completion_log=None, **kw):
    """trainer.py:409-414: continue training from an existing network."""
    return run_training(tiers, reward_spec, cfg, encoding=encoding, init_net=net,
                        completion_log=completion_log, **kw)
