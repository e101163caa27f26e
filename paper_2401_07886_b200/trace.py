"""Device-resident trace batches (WorkloadTrace, workload.py:39-91, as SoA).

Layout in HBM (env-major, row stride `ld`):
  arrival  f64 [E, ld]   task u8 [E, ld]   n_events i64 [E] (ragged rows)
  segments: CSR seg_offsets i64 [E+1] -> seg_start i64, seg_rate f64,
            seg_bucket i32 (reducer bucket per segment, optional)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .specs import ArrivalEvent, SegmentMark, WorkloadTrace


@dataclass
class TraceBatch:
    arrival: torch.Tensor
    task: torch.Tensor
    n_events: Optional[torch.Tensor]
    seg_offsets: torch.Tensor
    seg_start: torch.Tensor
    seg_rate: torch.Tensor
    seg_bucket: Optional[torch.Tensor] = None
    n_tasks: int = 0

    @property
    def n_envs(self) -> int:
        return int(self.arrival.shape[0])

    @property
    def ld(self) -> int:
        return int(self.arrival.shape[1])

    @property
    def device(self) -> torch.device:
        return self.arrival.device

    def soa(self) -> _lib.BeTraceSoa:
        s = _lib.BeTraceSoa()
        s.n_envs = self.n_envs
        s.ld = self.ld
        s.arrival_ms = self.arrival.data_ptr()
        s.task = self.task.data_ptr()
        s.n_events = _lib.ptr(self.n_events)
        s.seg_offsets = self.seg_offsets.data_ptr()
        s.seg_start = self.seg_start.data_ptr()
        s.seg_rate = self.seg_rate.data_ptr()
        s.seg_bucket = _lib.ptr(self.seg_bucket)
        return s

    def host_bytes(self) -> int:
        t = [self.arrival, self.task, self.n_events, self.seg_offsets, self.seg_start,
             self.seg_rate, self.seg_bucket]
        return sum(x.numel() * x.element_size() for x in t if x is not None)

    # ------------------------------------------------------------- builders
    @classmethod
    def from_arrays(cls, arrival: np.ndarray, task: np.ndarray, seg_start: Sequence,
                    seg_rate: Sequence, n_events=None, seg_bucket=None, device=None,
                    pin: bool = True) -> "TraceBatch":
        """arrival/task: [E, ld] (or [ld] for one env); seg_start/seg_rate: per-env
        sequences of SegmentMark start indices / rates."""
        dev = _lib.require_cuda(device)
        arrival = np.atleast_2d(np.asarray(arrival, np.float64))
        task = np.atleast_2d(np.asarray(task))
        if task.size and (not np.issubdtype(task.dtype, np.integer) or task.min() < 0 or task.max() > 255):
            raise _lib.InvalidParameterError("task ids must be integers in [0, 256)")
        task = task.astype(np.uint8)
        E = arrival.shape[0]
        if seg_start and np.ndim(seg_start[0]) == 0:
            seg_start, seg_rate = [seg_start], [seg_rate]
            if seg_bucket is not None:
                seg_bucket = [seg_bucket]
        offs = np.zeros(E + 1, np.int64)
        for e in range(E):
            offs[e + 1] = offs[e] + len(seg_start[e])
        ss = np.concatenate([np.asarray(s, np.int64) for s in seg_start]) if offs[-1] else np.zeros(0, np.int64)
        sr = np.concatenate([np.asarray(s, np.float64) for s in seg_rate]) if offs[-1] else np.zeros(0)
        sb = None
        if seg_bucket is not None:
            sb = np.concatenate([np.asarray(s, np.int32) for s in seg_bucket])
        _validate(arrival, n_events)

        def up(a):
            if a is None:
                return None
            t = torch.from_numpy(np.ascontiguousarray(a))
            if pin:
                t = t.pin_memory()
            return t.to(dev, non_blocking=True)

        return cls(arrival=up(arrival), task=up(task),
                   n_events=up(None if n_events is None else np.asarray(n_events, np.int64)),
                   seg_offsets=up(offs), seg_start=up(ss if ss.size else np.zeros(1, np.int64)),
                   seg_rate=up(sr if sr.size else np.zeros(1)), seg_bucket=up(sb),
                   n_tasks=int(task.max()) + 1 if task.size else 0)

    @classmethod
    def from_traces(cls, traces: Sequence, device=None, ld: Optional[int] = None,
                    buckets: Optional[Sequence[float]] = None) -> "TraceBatch":
        """Pack reference WorkloadTrace objects (one per env).  `buckets`: optional
        rate values; each segment maps to the nearest one (selection_distribution
        semantics, evalkit.py:255-258)."""
        lens = [len(t.events) for t in traces]
        ld = max(lens) if ld is None else ld
        E = len(traces)
        arr = np.zeros((E, max(ld, 1)), np.float64)
        tsk = np.zeros((E, max(ld, 1)), np.uint8)
        ss, sr, sb = [], [], []
        for e, tr in enumerate(traces):
            n = lens[e]
            if n:
                arr[e, :n] = [ev.time_ms for ev in tr.events]
                tsk[e, :n] = [ev.task_id for ev in tr.events]
            ss.append([m.start_index for m in tr.segment_marks])
            sr.append([m.rate for m in tr.segment_marks])
            if buckets is not None:
                b = np.asarray(buckets, float)
                sb.append([int(np.argmin(np.abs(b - m.rate))) for m in tr.segment_marks])
        ragged = any(n != ld for n in lens)
        return cls.from_arrays(arr, tsk, ss, sr, n_events=lens if ragged else None,
                               seg_bucket=sb if buckets is not None else None, device=device)

    @classmethod
    def generate_stable(cls, rates: Sequence[float], n: int, n_tasks: int, seed: int,
                        device=None, buckets: Optional[Sequence[int]] = None,
                        env_offset: int = 0) -> "TraceBatch":
        """On-device gen_stable (workload.py:120-141): env e is one Poisson
        segment at rates[e] req/s truncated to n requests (Philox4x32-10 keyed
        by (seed, env_offset + e), so a global env id gets the same trace on
        any number of GPUs)."""
        dev = _lib.require_cuda(device)
        E = len(rates)
        rate = torch.as_tensor(np.asarray(rates, np.float64), device=dev)
        arrival = torch.empty((E, n), dtype=torch.float64, device=dev)
        task = torch.empty((E, n), dtype=torch.uint8, device=dev)
        L = _lib.load()
        _lib.check(L.be_trace_gen_stable(E, int(env_offset), n, n, rate.data_ptr(), n_tasks, seed,
                                         arrival.data_ptr(), task.data_ptr(), _lib.stream_ptr()))
        offs = torch.arange(E + 1, dtype=torch.int64, device=dev)
        seg_start = torch.zeros(E, dtype=torch.int64, device=dev)
        sb = None if buckets is None else torch.as_tensor(np.asarray(buckets, np.int32), device=dev)
        return cls(arrival=arrival, task=task, n_events=None, seg_offsets=offs,
                   seg_start=seg_start, seg_rate=rate.clone(), seg_bucket=sb, n_tasks=n_tasks)

    @classmethod
    def generate(cls, workload: str, n_envs: int, n_tasks: int, seed: int, *,
                 n_requests: int = 10_000, rates: Optional[Sequence] = None,
                 hold_seconds: Optional[float] = None, task_ids: Optional[Sequence[int]] = None,
                 ld: Optional[int] = None, truncate: bool = False, seg_capacity: Optional[int] = None,
                 env_offset: int = 0, buckets: Optional[Sequence[float]] = None,
                 device=None) -> "TraceBatch":
        """On-device `make_trace` (evalkit.py:141-151) for `n_envs` environments.

        workload: "stable" (gen_stable, workload.py:120-141: `rates` — one list
        for every env or one list per env — each held `hold_seconds`),
        "unpredictable-time" (workload.py:144-171) or "unpredictable-request"
        (workload.py:174-198, `n_requests` each).  Draws are Philox4x32-10
        keyed by (seed, env_offset + e).  `truncate` keeps the first `ld`
        events of a stable trace (config 1); otherwise a stable trace longer
        than `ld` raises CapacityError.  `buckets`: optional rate values; each
        segment maps to the nearest (selection_distribution, evalkit.py:255-258)."""
        dev = _lib.require_cuda(device)
        if n_envs < 1:
            raise _lib.InvalidParameterError("n_envs must be >= 1")
        if n_tasks < 1:
            raise _lib.InvalidParameterError("n_tasks must be >= 1")
        cfg = _lib.BeGenCfg()
        cfg.n_tasks = n_tasks
        if task_ids is not None:
            ids = [int(t) for t in task_ids]
            if not ids or min(ids) < 0 or max(ids) >= n_tasks or len(ids) > _lib.MAX_TASKS:
                raise _lib.InvalidParameterError(f"task_ids must be a nonempty subset of [0, {n_tasks})")
            cfg.n_task_ids = len(ids)
            for k, t in enumerate(ids):
                cfg.task_ids[k] = t
        keep = None
        if workload == "stable":
            if rates is None or hold_seconds is None:
                raise _lib.InvalidParameterError("stable traces need rates and hold_seconds")
            r = np.asarray(rates, np.float64)
            if r.ndim == 1:
                r = r[None, :]
            if r.size == 0 or np.any(~(r > 0)) or not np.all(np.isfinite(r)):
                raise _lib.InvalidParameterError("rates must be nonempty and positive")
            if not hold_seconds > 0:
                raise _lib.InvalidParameterError("hold_seconds must be positive")
            if r.shape[0] not in (1, n_envs):
                raise ValueError("rates: one row for every env or one row per env")
            keep = torch.as_tensor(np.ascontiguousarray(r), device=dev)
            cfg.kind = _lib.GEN_STABLE
            cfg.n_rates = r.shape[1]
            cfg.rate_ld = 0 if r.shape[0] == 1 else r.shape[1]
            cfg.rates = keep.data_ptr()
            cfg.hold_ms = float(hold_seconds) * 1000.0
            cfg.truncate = 1 if truncate else 0
            if ld is None:  # expected count + 8 sigma + slack
                lam = float(np.max(r.sum(axis=1))) * float(hold_seconds)
                ld = int(lam + 8.0 * np.sqrt(lam) + 64)
            seg_capacity = seg_capacity or r.shape[1]
        elif workload in ("unpredictable-time", "unpredictable-request"):
            if n_requests < 1:
                raise _lib.InvalidParameterError("n_requests must be >= 1")
            cfg.kind = _lib.GEN_UNPRED_TIME if workload == "unpredictable-time" else _lib.GEN_UNPRED_REQ
            cfg.n = n_requests
            ld = n_requests if ld is None else ld
            # expected segments: ~1/70 (time-based) or 1/500 (request-based) of the requests
            seg_capacity = seg_capacity or max(64, n_requests // 8 + 64)
        else:
            raise ValueError(f"unknown workload kind {workload!r}")
        cfg.seg_capacity = seg_capacity
        E = n_envs
        arrival = torch.empty((E, ld), dtype=torch.float64, device=dev)
        task = torch.zeros((E, ld), dtype=torch.uint8, device=dev)
        n_events = torch.empty(E, dtype=torch.int64, device=dev)
        seg_count = torch.empty(E, dtype=torch.int64, device=dev)
        ss = torch.empty((E, seg_capacity), dtype=torch.int64, device=dev)
        sr = torch.empty((E, seg_capacity), dtype=torch.float64, device=dev)
        status = torch.zeros(2, dtype=torch.int32, device=dev)
        L = _lib.load()
        _lib.check(L.be_trace_gen(ctypes.byref(cfg), E, int(env_offset), ld, seed & (2**64 - 1),
                                  arrival.data_ptr(), task.data_ptr(), n_events.data_ptr(),
                                  seg_count.data_ptr(), ss.data_ptr(), sr.data_ptr(),
                                  status.data_ptr(), _lib.stream_ptr()))
        st = status.cpu().tolist()
        if st[0] == _lib.BE_ECAPACITY:
            raise _lib.CapacityError(f"env {st[1]}: trace exceeds ld={ld} events or "
                                     f"seg_capacity={seg_capacity} segments")
        if st[0] != 0:
            raise _lib.InvalidParameterError(f"env {st[1]}: invalid generator parameters")
        # pad ragged rows with their last arrival so every row stays sorted
        col = torch.arange(ld, device=dev)
        last = arrival.gather(1, (n_events - 1).clamp(min=0)[:, None])
        arrival = torch.where(col[None, :] < n_events[:, None], arrival, last)
        # segment marks -> CSR
        sel = torch.arange(seg_capacity, device=dev)[None, :] < seg_count[:, None]
        offs = torch.zeros(E + 1, dtype=torch.int64, device=dev)
        offs[1:] = torch.cumsum(seg_count, 0)
        seg_start, seg_rate = ss[sel], sr[sel]
        sb = None
        if buckets is not None:
            b = torch.as_tensor(np.asarray(buckets, np.float64), device=dev)
            sb = torch.argmin((seg_rate[:, None] - b[None, :]).abs(), dim=1).to(torch.int32)
        ragged = bool((n_events != ld).any())
        return cls(arrival=arrival, task=task, n_events=n_events if ragged else None,
                   seg_offsets=offs, seg_start=seg_start if seg_start.numel() else
                   torch.zeros(1, dtype=torch.int64, device=dev),
                   seg_rate=seg_rate if seg_rate.numel() else torch.zeros(1, device=dev, dtype=torch.float64),
                   seg_bucket=sb, n_tasks=n_tasks)

    @classmethod
    def from_scenario(cls, scenario, n_envs: int, n_tasks: int, seed: int, *, env_offset: int = 0,
                      device=None, **kw) -> "TraceBatch":
        """`make_trace(scenario, n_tasks, seed)` (evalkit.py:141-151) for n_envs envs
        on the device.  `scenario`: a ScenarioConfig-like object (workload, rates,
        hold_seconds, n_requests, task_ids) or a scenario name."""
        if isinstance(scenario, str):
            from .evalkit import scenario_suite
            scenario = scenario_suite(scenario)
        kind = {"stable": "stable", "unpredictable-time": "unpredictable-time",
                "unpredictable-request": "unpredictable-request"}.get(scenario.workload)
        if kind is None:
            raise ValueError(f"unknown workload kind {scenario.workload!r}")
        return cls.generate(kind, n_envs, n_tasks, seed, n_requests=scenario.n_requests,
                            rates=scenario.rates, hold_seconds=scenario.hold_seconds,
                            task_ids=scenario.task_ids, env_offset=env_offset, device=device, **kw)

    # ------------------------------------------------------------- export
    def to_workload_trace(self, e: int, seed: int = 0) -> WorkloadTrace:
        """Env e as a WorkloadTrace (replayable by the reference's run_eval)."""
        n = self.ld if self.n_events is None else int(self.n_events[e])
        arr = self.arrival[e, :n].cpu().numpy()
        tsk = self.task[e, :n].cpu().numpy()
        o0, o1 = int(self.seg_offsets[e]), int(self.seg_offsets[e + 1])
        ss = self.seg_start[o0:o1].cpu().numpy()
        sr = self.seg_rate[o0:o1].cpu().numpy()
        return WorkloadTrace(events=[ArrivalEvent(float(t), int(k)) for t, k in zip(arr, tsk)],
                             segment_marks=[SegmentMark(int(a), float(b)) for a, b in zip(ss, sr)],
                             seed=seed)

    def event_rates(self, e: int) -> np.ndarray:
        n = self.ld if self.n_events is None else int(self.n_events[e])
        o0, o1 = int(self.seg_offsets[e]), int(self.seg_offsets[e + 1])
        ss = self.seg_start[o0:o1].cpu().numpy()
        sr = self.seg_rate[o0:o1].cpu().numpy()
        out = np.full(n, np.nan)
        for k in range(len(ss)):
            end = ss[k + 1] if k + 1 < len(ss) else n
            out[ss[k]:end] = sr[k]
        return out


def _validate(arrival: np.ndarray, n_events) -> None:
    """WorkloadTrace.validate / RateEstimator.observe ordering (workload.py:61-72, :235-237)."""
    E, ld = arrival.shape
    if ld > (1 << 24):
        raise _lib.InvalidParameterError("traces longer than 2^24 requests are not supported")
    for e in range(E):
        n = ld if n_events is None else int(n_events[e])
        a = arrival[e, :n]
        if n and (not np.all(np.isfinite(a)) or a[0] < 0 or np.any(np.diff(a) < 0)):
            raise ValueError(f"env {e}: arrival times must be finite, nonnegative and sorted")
