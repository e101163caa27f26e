"""Greedy rollout + evaluation on the GPU (drop-ins for besteffort.evalkit).

  run_eval            evalkit.py:154-209  (same signature, same EvalRun records)
  run_eval_batch      the same loop for E envs in one persistent kernel
  windowed / threshold_counts / miss fractions   evalkit.py:212-241, :61-74
                      -> be_reduce_eval (sequential fp64 scan per env on device)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .env import EnvBatch, default_ring_capacity
from .policy import DeviceQNet
from .specs import StateEncoding, event_rates
from .trace import TraceBatch

WINDOW = 20
THRESHOLDS = (1.00, 0.99, 0.98, 0.96, 0.94)
PAPER_THRESHOLDS = (1.00, 0.98, 0.96, 0.94, 0.90)  # north-star: >= 90/94/96/98% of peak
STABLE_SWEEP_RATES = (0.25, 0.5, 1.0, 2.0, 3.0, 4.0, 6.0, 8.0, 12.0, 16.0, 24.0, 32.0, 40.0, 48.0)
STABLE_HOLD_SECONDS = 40.0


@dataclass(frozen=True)
class ScenarioConfig:
    """evalkit.py:77-102 (host-side configuration, same fields and semantics)."""
    name: str
    workload: str = "stable"  # stable | unpredictable-time | unpredictable-request
    rates: tuple = STABLE_SWEEP_RATES
    hold_seconds: float = STABLE_HOLD_SECONDS
    n_requests: int = 10_000
    task_ids: Optional[tuple] = None
    estimator_mode: str = "estimated"
    reset_between_segments: bool = False
    reward_kind: Optional[str] = None
    deadline_overrides: tuple = ()
    replicas: Optional[int] = None
    gpu_count: Optional[int] = None

    def adjust_rewards(self, spec):
        if self.reward_kind is not None:
            spec = spec.with_kind(self.reward_kind)
        if self.deadline_overrides:
            spec = spec.with_deadlines(dict(self.deadline_overrides))
        return spec

    def adjust_tiers(self, tiers):
        if self.replicas is None:
            return list(tiers)
        from dataclasses import replace
        return [replace(t, replicas=self.replicas) for t in tiers]


_SCENARIOS = {  # evalkit.py:105-131
    "stable": ScenarioConfig(name="stable", workload="stable", estimator_mode="true-rate",
                             reset_between_segments=True),
    "unpredictable-1": ScenarioConfig(name="unpredictable-1", workload="unpredictable-time"),
    "unpredictable-2": ScenarioConfig(name="unpredictable-2", workload="unpredictable-request"),
    "hellaswag-copa-soft": ScenarioConfig(name="hellaswag-copa-soft", workload="unpredictable-time",
                                          task_ids=(0, 1), reward_kind="soft"),
    "different-deadlines": ScenarioConfig(name="different-deadlines", workload="stable",
                                          estimator_mode="true-rate", reset_between_segments=True,
                                          deadline_overrides=(("openbookqa", 80.0), ("copa", 32.0))),
    "hw-utility-8gpu": ScenarioConfig(name="hw-utility-8gpu", workload="unpredictable-time",
                                      replicas=8, gpu_count=8),
}
for _k in range(4):
    _SCENARIOS[f"single-task-{_k}"] = ScenarioConfig(
        name=f"single-task-{_k}", workload="stable", estimator_mode="true-rate",
        reset_between_segments=True, task_ids=(_k,))


def scenario_names() -> list:
    return sorted(_SCENARIOS)


def scenario_suite(name: str) -> ScenarioConfig:
    """evalkit.py:134-138."""
    try:
        return _SCENARIOS[name]
    except KeyError:
        raise ValueError(f"unknown scenario {name!r}; known: {', '.join(scenario_names())}")


@dataclass
class RequestRecord:
    index: int
    arrival_ms: float
    task_id: int
    tier_id: int
    reward: float
    realized_ms_per_token: float
    segment_rate: float


@dataclass
class EvalRun:
    records: list
    policy_id: str
    gpu_count: int
    seed: int

    def rewards(self) -> np.ndarray:
        return np.array([r.reward for r in self.records])

    def rates(self) -> np.ndarray:
        return np.array([r.segment_rate for r in self.records])

    def miss_fractions_by_rate(self, spec) -> dict:
        missed: dict = {}
        for r in self.records:
            deadline = spec.tasks[r.task_id].deadline_ms_per_token
            missed.setdefault(r.segment_rate, []).append(
                1 if r.realized_ms_per_token > deadline else 0)
        return {rate: float(np.mean(v)) for rate, v in missed.items()}

    def mean_reward_by_rate(self) -> dict:
        by_rate: dict = {}
        for r in self.records:
            by_rate.setdefault(r.segment_rate, []).append(r.reward)
        return {rate: float(np.mean(v)) for rate, v in by_rate.items()}


@dataclass
class RolloutOutputs:
    flags: torch.Tensor            # u8 [E, ld]: tier | miss << 7
    reward: torch.Tensor           # f64 [E, ld]
    realized: Optional[torch.Tensor] = None
    obs: Optional[torch.Tensor] = None    # i32 [E, ld, M]
    rate: Optional[torch.Tensor] = None   # f64 [E, ld]
    q: Optional[torch.Tensor] = None      # f64 [E, ld, M]

    @property
    def tier(self) -> torch.Tensor:
        return self.flags & 0x3F  # bit 6 = completed, bit 7 = deadline miss

    @property
    def miss(self) -> torch.Tensor:
        return (self.flags >> 7).to(torch.bool)


class GreedyRollout:
    """Reusable fused rollout for trace batches of a fixed shape.

    Owns the env handle (replica rings) and the output buffers, so repeated
    runs allocate nothing.  Every run re-initialises the envs in-kernel.

    ring_capacity=None ("auto"): the per-replica FIFO rings start small
    (AUTO_RING_START slots, so the rings of the envs in flight stay resident in
    L2) and `run` grows them 4x and re-runs when a ring overflows — overflow is
    always detected on the device; results do not depend on the capacity."""

    AUTO_RING_START = 64

    def __init__(self, tiers, reward_spec, n_envs: int, ld: int, encoding=None, *,
                 estimator_mode: str = "estimated", prior_rate: float = 1.0,
                 reset_between_segments: bool = False, ring_capacity: Optional[int] = None,
                 skip_ahead: bool = True, want_realized: bool = True, want_steps: bool = False,
                 q_screen: bool = True, device=None):
        self.device = _lib.require_cuda(device)
        R = sum(int(t.replicas) for t in tiers)
        self._auto_ring = ring_capacity is None
        if ring_capacity is None:
            free, _ = torch.cuda.mem_get_info(self.device)
            self._ring_max = default_ring_capacity(ld, n_envs, R, budget_bytes=int(free * 0.35))
            ring_capacity = min(self._ring_max, self.AUTO_RING_START)
        else:
            self._ring_max = int(ring_capacity)
        self._env_args = (tiers, reward_spec, n_envs, encoding)
        self._env_kw = dict(estimator_mode=estimator_mode, prior_rate=prior_rate,
                            reset_between_segments=reset_between_segments, skip_ahead=skip_ahead,
                            q_screen=q_screen, device=self.device)
        self.env = EnvBatch(*self._env_args, ring_capacity=ring_capacity, **self._env_kw)
        self.n_envs, self.ld, self.M = int(n_envs), int(ld), len(tiers)
        dev = self.device
        self.out = RolloutOutputs(
            flags=torch.zeros((n_envs, ld), dtype=torch.uint8, device=dev),
            reward=torch.zeros((n_envs, ld), dtype=torch.float64, device=dev),
            realized=torch.zeros((n_envs, ld), dtype=torch.float64, device=dev) if want_realized else None,
            obs=torch.zeros((n_envs, ld, self.M), dtype=torch.int32, device=dev) if want_steps else None,
            rate=torch.zeros((n_envs, ld), dtype=torch.float64, device=dev) if want_steps else None,
            q=torch.zeros((n_envs, ld, self.M), dtype=torch.float64, device=dev) if want_steps else None)

    @property
    def ring_capacity(self) -> int:
        return self.env.ring_capacity

    def _grow_ring(self) -> bool:
        cap = self.env.ring_capacity
        if not self._auto_ring or cap >= self._ring_max:
            return False
        self.env.close()
        self.env = EnvBatch(*self._env_args, ring_capacity=min(self._ring_max, cap * 4), **self._env_kw)
        return True

    def launch(self, trace: TraceBatch, policy=None, static_tier: int = -1,
               forced: Optional[torch.Tensor] = None, stream=None, ready=None) -> RolloutOutputs:
        """Asynchronous: enqueue the fused rollout on `stream` (no sync)."""
        if trace.n_envs > self.n_envs or trace.ld != self.ld:
            raise ValueError("trace batch does not match the rollout shape")
        if trace.n_tasks > self.env.n_tasks:  # the kernel also flags ids >= n_tasks (EINVAL)
            raise ValueError(f"trace task ids reach {trace.n_tasks - 1}, the reward spec has "
                             f"{self.env.n_tasks} tasks")
        o = self.out
        rec = _lib.BeRecords()
        rec.flags, rec.reward = o.flags.data_ptr(), o.reward.data_ptr()
        rec.realized = _lib.ptr(o.realized)
        rec.obs, rec.rate = _lib.ptr(o.obs), _lib.ptr(o.rate)
        rec.q = _lib.ptr(o.q) if (policy is not None and static_tier < 0 and forced is None) else None
        w = None
        if forced is None and static_tier < 0:
            if policy is None:
                raise ValueError("need a policy, a static tier or forced actions")
            self._dn = DeviceQNet.of(policy, self.device)
            w = self._dn.weights()
        soa = trace.soa()
        if ready is not None:  # streamed upload (StreamingEvaluator): per-chunk ready flags
            flags, per, value = ready
            soa.env_ready, soa.envs_per_ready, soa.ready_value = flags.data_ptr(), int(per), int(value)
        _lib.check(self.env._L.be_rollout_greedy(self.env.handle, soa, w, int(static_tier),
                                                 _lib.ptr(forced), rec, _lib.stream_ptr(stream)))
        return o

    def run(self, trace: TraceBatch, policy=None, static_tier: int = -1,
            forced: Optional[torch.Tensor] = None, stream=None) -> RolloutOutputs:
        """Synchronous rollout; with an "auto" ring it grows and re-runs on overflow."""
        while True:
            o = self.launch(trace, policy, static_tier, forced, stream)
            try:
                self.env.check(stream)  # sync + raise on ring overflow / bad action
                return o
            except _lib.CapacityError:
                if not self._grow_ring():
                    raise


def _policy_args(policy, n_tiers):
    if isinstance(policy, (int, np.integer)) and not isinstance(policy, bool):
        st = int(policy)
        if not 0 <= st < n_tiers:
            raise ValueError(f"static tier {st} out of range")
        return None, st
    return policy, -1


def run_eval(policy, trace, tiers, reward_spec, encoding=None, seed: int = 0, *,
             gpu_count: int = 4, estimator_mode: str = "estimated", prior_rate: float = 1.0,
             reset_between_segments: bool = False, policy_id: Optional[str] = None,
             device=None) -> EvalRun:
    """Drop-in for besteffort.evalkit.run_eval (evalkit.py:154-209), on the GPU."""
    net, static_tier = _policy_args(policy, len(tiers))
    if static_tier < 0 and encoding is None:
        encoding = StateEncoding(n_tasks=len(reward_spec.tasks),
                                 batch_scales=tuple(float(t.max_batch) for t in tiers))
    if policy_id is None:
        policy_id = f"static:{static_tier}" if static_tier >= 0 else "policy"
    tb = TraceBatch.from_traces([trace], device=device)
    ro = GreedyRollout(tiers, reward_spec, 1, tb.ld, encoding, estimator_mode=estimator_mode,
                       prior_rate=prior_rate, reset_between_segments=reset_between_segments,
                       device=device)
    o = ro.run(tb, net, static_tier)
    n = len(trace.events)
    tier = o.tier[0, :n].cpu().numpy()
    rw = o.reward[0, :n].cpu().numpy()
    rl = o.realized[0, :n].cpu().numpy()
    rates = event_rates(trace)
    records = [RequestRecord(i, ev.time_ms, ev.task_id, int(tier[i]), float(rw[i]), float(rl[i]),
                             float(rates[i])) for i, ev in enumerate(trace.events)]
    return EvalRun(records=records, policy_id=policy_id, gpu_count=gpu_count, seed=seed)


# --------------------------------------------------------------- reducer
@dataclass
class ReduceResult:
    thresholds: tuple
    win_counts: torch.Tensor     # i64 [E, n_theta]
    n_windows: torch.Tensor      # i64 [E]
    bucket_miss: torch.Tensor    # i64 [E, K]
    bucket_req: torch.Tensor     # i64 [E, K]
    bucket_reward: torch.Tensor  # f64 [E, K] (sequential per env)

    def totals(self) -> dict:
        """Whole-batch stats (int64 sums are exact; reward sums in env order)."""
        wc = self.win_counts.sum(0).cpu().numpy()
        nw = int(self.n_windows.sum())
        miss = self.bucket_miss.sum(0).cpu().numpy()
        req = self.bucket_req.sum(0).cpu().numpy()
        rws = self.bucket_reward.cpu().numpy().sum(0)
        with np.errstate(invalid="ignore", divide="ignore"):
            return dict(
                thresholds=list(self.thresholds), win_counts=wc.tolist(), n_windows=nw,
                window_fraction=(wc / max(nw, 1)).tolist(),
                requests=req.tolist(), misses=miss.tolist(),
                availability=(1.0 - miss / np.maximum(req, 1)).tolist(),
                mean_reward=(rws / np.maximum(req, 1)).tolist())


def reduce_eval(trace: TraceBatch, flags: torch.Tensor, reward: torch.Tensor,
                thresholds: Sequence[float] = THRESHOLDS, n_buckets: int = 1,
                window: int = WINDOW, stream=None) -> ReduceResult:
    """On-device windowed + threshold_counts + per-bucket miss/request/reward."""
    E, dev = trace.n_envs, trace.device
    if not 1 <= len(thresholds) <= _lib.MAX_THETA:
        raise ValueError(f"between 1 and {_lib.MAX_THETA} thresholds")
    th = _lib.BeThresholds()
    th.n = len(thresholds)
    for k, t in enumerate(thresholds):
        th.theta[k] = float(t)
    K = int(n_buckets)
    out = ReduceResult(tuple(thresholds),
                       torch.empty((E, len(thresholds)), dtype=torch.int64, device=dev),
                       torch.empty(E, dtype=torch.int64, device=dev),
                       torch.empty((E, K), dtype=torch.int64, device=dev),
                       torch.empty((E, K), dtype=torch.int64, device=dev),
                       torch.empty((E, K), dtype=torch.float64, device=dev))
    L = _lib.load()
    _lib.check(L.be_reduce_eval(trace.soa(), flags.data_ptr(), reward.data_ptr(), int(window),
                                th, K, out.win_counts.data_ptr(),
                                out.n_windows.data_ptr(), out.bucket_miss.data_ptr(),
                                out.bucket_req.data_ptr(), out.bucket_reward.data_ptr(),
                                _lib.stream_ptr(stream)))
    return out


class StreamingEvaluator:
    """End-to-end evaluation of host-resident trace batches.

    Each `submit` copies one pinned-host trace batch to the device on a copy
    stream (double-buffered, so batch k+1 uploads while batch k rolls out),
    runs the fused rollout + reducer on the compute stream and copies the
    int64 / f64 statistics back.  `result(k)` waits for batch k."""

    def __init__(self, policy, tiers, reward_spec, n_envs: int, ld: int, encoding=None, *,
                 estimator_mode: str = "estimated", thresholds=THRESHOLDS, n_buckets: int = 1,
                 ring_capacity: Optional[int] = None, device=None):
        self.device = _lib.require_cuda(device)
        self.net, self.static_tier = _policy_args(policy, len(tiers))
        if self.static_tier < 0 and encoding is None:
            encoding = StateEncoding(n_tasks=len(reward_spec.tasks),
                                     batch_scales=tuple(float(t.max_batch) for t in tiers))
        if ring_capacity is None:  # double-buffered: no re-run on overflow, size for the worst case
            free, _ = torch.cuda.mem_get_info(self.device)
            ring_capacity = default_ring_capacity(ld, n_envs, sum(int(t.replicas) for t in tiers),
                                                  budget_bytes=int(free * 0.35))
        self.ro = GreedyRollout(tiers, reward_spec, n_envs, ld, encoding,
                                estimator_mode=estimator_mode, ring_capacity=ring_capacity,
                                want_realized=False, device=self.device)
        if self.net is not None:
            self.net = DeviceQNet.of(self.net, self.device)
        self.thresholds, self.n_buckets = tuple(thresholds), int(n_buckets)
        self.copy_stream = torch.cuda.Stream(self.device)
        self.compute_stream = torch.cuda.Stream(self.device)
        self._bufs = [None, None]
        self._copied = [torch.cuda.Event(), torch.cuda.Event()]
        self._freed = [torch.cuda.Event(), torch.cuda.Event()]
        self._k = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # pinned host buffers for the statistics, allocated up front (pinned allocation
        # synchronises the device): up to `max_outstanding` submits may await result()
        self._stat_pool = []
        self._stat_shapes = None
        self.max_outstanding = 8
        self._flags = None

    def _device_buf(self, slot: int, host: TraceBatch) -> TraceBatch:
        b = self._bufs[slot]
        if b is None:
            def like(t):
                return None if t is None else torch.empty_like(t, device=self.device)
            b = TraceBatch(like(host.arrival), like(host.task), like(host.n_events),
                           like(host.seg_offsets), like(host.seg_start), like(host.seg_rate),
                           like(host.seg_bucket), host.n_tasks)
            self._bufs[slot] = b
        return b

    CHUNKS = 16  # streamed upload: the rollout starts once the first 1/16 of the envs arrived

    def submit(self, host: TraceBatch):
        """host: a TraceBatch whose tensors live in pinned host memory.

        The small per-env / per-segment arrays are copied first; the arrival and
        task rows follow in CHUNKS env ranges, each followed by a 4-byte copy that
        sets its ready flag, and the rollout (launched right after the metadata)
        waits per env for its chunk's flag (be_trace_soa.env_ready) — so the
        rollout of the first envs overlaps the upload of the rest."""
        slot = self._k & 1
        dev = self._device_buf(slot, host)
        cs, ks = self.copy_stream, self.compute_stream
        E = host.n_envs
        per = max(1, -(-E // self.CHUNKS))
        n_chunks = -(-E // per)
        if self._flags is None:
            self._flags = [torch.zeros(self.CHUNKS, dtype=torch.int32, device=self.device) for _ in range(2)]
            self._flag_vals = torch.arange(1, 1 << 16, dtype=torch.int32).pin_memory()
        value = (self._k // 2) % (self._flag_vals.numel()) + 1  # per slot: 1, 2, 3, ... then wraps
        flags = self._flags[slot]
        with torch.cuda.stream(cs):
            cs.wait_event(self._freed[slot])  # previous use of this buffer finished
            if value == 1:
                flags.zero_()  # first use of the slot, or the value wrapped: flags below 1 again
            nbytes = 0
            for name in ("n_events", "seg_offsets", "seg_start", "seg_rate", "seg_bucket"):
                src, dst = getattr(host, name), getattr(dev, name)
                if src is not None:
                    dst.copy_(src, non_blocking=True)
                    nbytes += src.numel() * src.element_size()
            self._copied[slot].record(cs)
            for c in range(n_chunks):
                lo, hi = c * per, min(E, (c + 1) * per)
                for name in ("arrival", "task"):
                    src, dst = getattr(host, name), getattr(dev, name)
                    dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                    nbytes += src[lo:hi].numel() * src.element_size()
                flags[c:c + 1].copy_(self._flag_vals[value - 1:value], non_blocking=True)
        self.h2d_bytes = nbytes
        with torch.cuda.stream(ks):
            ks.wait_event(self._copied[slot])
            o = self.ro.launch(dev, self.net, self.static_tier, stream=ks,
                               ready=(flags, per, value))
            red = reduce_eval(dev, o.flags, o.reward, self.thresholds, self.n_buckets, stream=ks)
            self._freed[slot].record(ks)
            host_stats = self._stats_buffer(red)
            for k, t in host_stats.items():
                if k != "status":
                    t.copy_(getattr(red, k), non_blocking=True)
            # the env's latched status rides with the statistics: result() needs no
            # stream-wide synchronisation (which would also wait for the next batch)
            _lib.check(self.ro.env._L.be_env_status_async(self.ro.env.handle, host_stats["status"].data_ptr(),
                                                           _lib.stream_ptr(ks)))
            done = torch.cuda.Event()
            done.record(ks)
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in host_stats.values())
        self._k += 1
        return done, host_stats

    _STATS = ("win_counts", "n_windows", "bucket_miss", "bucket_req", "bucket_reward")

    def _stats_buffer(self, red) -> dict:
        shapes = tuple((tuple(getattr(red, k).shape), getattr(red, k).dtype) for k in self._STATS)
        if shapes != self._stat_shapes:
            self._stat_shapes = shapes
            self._stat_pool = [dict({k: torch.empty(sh, dtype=dt, pin_memory=True)
                                     for k, (sh, dt) in zip(self._STATS, shapes)},
                                    status=torch.zeros(2, dtype=torch.int32, pin_memory=True))
                               for _ in range(self.max_outstanding)]
        if not self._stat_pool:
            raise RuntimeError(f"more than {self.max_outstanding} submits await result()")
        return self._stat_pool.pop()

    def result(self, handle) -> ReduceResult:
        done, hs = handle
        done.synchronize()
        if int(hs["status"][0]) != 0:  # raise with the library's message (syncs, error path only)
            self._stat_pool.append(hs)
            self.ro.env.check(self.compute_stream)
        out = ReduceResult(self.thresholds, *(hs[k].clone() for k in self._STATS))
        self._stat_pool.append(hs)
        return out


def pin_trace(tb: TraceBatch) -> TraceBatch:
    """Copy a device TraceBatch into pinned host memory (for end-to-end runs)."""
    def h(t):
        return None if t is None else t.cpu().pin_memory()
    return TraceBatch(h(tb.arrival), h(tb.task), h(tb.n_events), h(tb.seg_offsets),
                      h(tb.seg_start), h(tb.seg_rate), h(tb.seg_bucket), tb.n_tasks)


def run_eval_batch(policy, traces: Union[TraceBatch, Sequence], tiers, reward_spec, encoding=None,
                   *, estimator_mode: str = "estimated", prior_rate: float = 1.0,
                   reset_between_segments: bool = False, thresholds=THRESHOLDS,
                   buckets: Optional[Sequence[float]] = None, ring_capacity: Optional[int] = None,
                   device=None):
    """run_eval over many envs at once + the on-device reducer.
    Returns (RolloutOutputs, ReduceResult)."""
    net, static_tier = _policy_args(policy, len(tiers))
    if static_tier < 0 and encoding is None:
        encoding = StateEncoding(n_tasks=len(reward_spec.tasks),
                                 batch_scales=tuple(float(t.max_batch) for t in tiers))
    tb = traces if isinstance(traces, TraceBatch) else TraceBatch.from_traces(
        list(traces), device=device, buckets=buckets)
    ro = GreedyRollout(tiers, reward_spec, tb.n_envs, tb.ld, encoding,
                       estimator_mode=estimator_mode, prior_rate=prior_rate,
                       reset_between_segments=reset_between_segments,
                       ring_capacity=ring_capacity, device=device)
    o = ro.run(tb, net, static_tier)
    K = 1 if buckets is None else len(buckets)
    red = reduce_eval(tb, o.flags, o.reward, thresholds, K)
    return o, red


# --------------------------------------------------------------- secondary reducers
# evalkit.py:212-297.  The per-request work (selection counts, windowed series)
# runs on the device; the O(K) post-processing mirrors the reference on the host.

def bucket_segments(trace: TraceBatch, rate_buckets: Sequence[float]) -> TraceBatch:
    """Map every segment to the nearest rate bucket (first minimum, like the
    np.argmin in selection_distribution, evalkit.py:257) -> trace.seg_bucket."""
    b = torch.as_tensor(np.asarray(rate_buckets, np.float64), device=trace.device)
    trace.seg_bucket = torch.argmin((trace.seg_rate[:, None] - b[None, :]).abs(), dim=1).to(torch.int32)
    return trace


def selection_counts(trace: TraceBatch, flags: torch.Tensor, n_tasks: int, n_tiers: int,
                     n_buckets: int, stream=None) -> torch.Tensor:
    """int64 [T, K, M] request counts per (task, rate bucket, tier) over all envs
    (be_reduce_selection; buckets from trace.seg_bucket)."""
    counts = torch.zeros((n_tasks, n_buckets, n_tiers), dtype=torch.int64, device=trace.device)
    L = _lib.load()
    _lib.check(L.be_reduce_selection(trace.soa(), flags.data_ptr(), int(n_tasks), int(n_tiers),
                                     int(n_buckets), counts.data_ptr(), _lib.stream_ptr(stream)))
    return counts


def selection_distribution(runs, rate_buckets: Sequence[float], n_tasks: int, n_tiers: int,
                           flags: Optional[torch.Tensor] = None) -> np.ndarray:
    """evalkit.py:244-262: tier-selection frequency per (task, rate bucket), (T, K, M).

    `runs`: a TraceBatch (with `flags` = RolloutOutputs.flags of its rollout — the
    counting runs on the device), or a sequence of EvalRun (reference or ours)."""
    buckets = np.asarray(rate_buckets, dtype=float)
    if isinstance(runs, TraceBatch):
        if flags is None:
            raise ValueError("need the rollout flags for a TraceBatch")
        bucket_segments(runs, buckets)
        counts = selection_counts(runs, flags, n_tasks, n_tiers, buckets.size).cpu().numpy().astype(float)
    else:
        if not runs:
            raise ValueError("need at least one run")
        counts = np.zeros((n_tasks, buckets.size, n_tiers))
        for run in runs:
            for r in run.records:
                k = int(np.argmin(np.abs(buckets - r.segment_rate)))
                counts[r.task_id, k, r.tier_id] += 1
    totals = counts.sum(axis=2, keepdims=True)
    with np.errstate(invalid="ignore"):
        return np.where(totals > 0, counts / np.maximum(totals, 1), 0.0)


def riemann_usage(freq: np.ndarray, rate_buckets: Sequence[float], task_id: int, tier_id: int) -> float:
    """evalkit.py:265-270: left-endpoint Riemann sum over the sweep."""
    rates = np.asarray(rate_buckets, dtype=float)
    return float(np.sum(freq[task_id, :-1, tier_id] * np.diff(rates)))


def hardware_utility(run_or_rewards, gpu_count: int):
    """evalkit.py:273-277: per-request reward / GPUs backing the system."""
    if gpu_count < 1:
        raise ValueError("gpu_count must be >= 1")
    r = run_or_rewards.rewards() if hasattr(run_or_rewards, "rewards") else run_or_rewards
    return r / gpu_count


def trial_band(series):
    """evalkit.py:280-288: pointwise mean and population std across trials."""
    if len(series) < 2:
        raise ValueError("need at least two runs")
    if isinstance(series, torch.Tensor):
        return series.mean(dim=0), series.std(dim=0, unbiased=False)
    if len({len(s) for s in series}) != 1:
        raise ValueError("runs must have equal length")
    stack = np.asarray(series, dtype=float)
    return stack.mean(axis=0), stack.std(axis=0)


def collapse_rate(miss_by_rate: dict, rates: Sequence[float], threshold: float = 0.5):
    """evalkit.py:291-297: lowest swept rate whose miss fraction exceeds threshold."""
    for rate in rates:
        if miss_by_rate.get(rate, 0.0) > threshold:
            return float(rate)
    return None


def running_average(values) -> np.ndarray:
    """evalkit.py:212-214."""
    v = np.asarray(values, dtype=float)
    return np.cumsum(v) / np.arange(1, v.size + 1)


def windowed(trace: TraceBatch, reward: torch.Tensor, window: int = WINDOW, stream=None) -> torch.Tensor:
    """evalkit.py:217-226 for every env on the device: f64 [E, ld]; row e holds its
    n_e - window + 1 trailing means first (bit-identical to the reference)."""
    if window < 1:
        raise ValueError("window must be >= 1")
    out = torch.full((trace.n_envs, trace.ld), float("nan"), dtype=torch.float64, device=trace.device)
    L = _lib.load()
    _lib.check(L.be_windowed(trace.soa(), reward.data_ptr(), int(window), out.data_ptr(),
                             _lib.stream_ptr(stream)))
    return out
