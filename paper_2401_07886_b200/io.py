"""Byte-identical CSV I/O of the reference, host side.

  write_trace / read_trace       workload.py:258-321 (`# rng`, `# seed`, `# segment`
                                 comment lines, repr floats, validating reader)
  write_metrics_csv / read_...   evalkit.py:300-321 (7-column per-request CSV)
  summary_row / write_summary    cli.py:145-160, :184-195 (threshold-window counts)
  write_per_rate                 cli.py:203-216

The GPU rollout fills EvalRun records (evalkit.run_eval / run_eval_batch ->
records); these writers produce the same bytes the reference CLI writes for the
same records (tests/test_io_cpu.py pins them against reference-written files).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from ._lib import InvalidParameterError
from .specs import RNG_ALGO, ArrivalEvent, SegmentMark, WorkloadTrace

METRICS_HEADER = "request_index,arrival_ms,task_id,tier_id,reward,realized_ms_per_token,segment_rate"
THRESHOLDS = (1.00, 0.99, 0.98, 0.96, 0.94)


class TraceParseError(InvalidParameterError):
    """workload.py:32-36: a malformed trace file, with path and line number."""

    def __init__(self, message: str, path: str, lineno: int):
        super().__init__(f"{path}:{lineno}: {message}")
        self.path = path
        self.lineno = lineno


def write_trace(trace, path: str) -> None:
    """workload.py:258-267."""
    if hasattr(trace, "validate"):
        trace.validate()
    rng_algo = getattr(trace, "rng_algo", RNG_ALGO)
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(f"# rng,{rng_algo}\n")
        f.write(f"# seed,{trace.seed}\n")
        for mark in trace.segment_marks:
            f.write(f"# segment,{mark.start_index},{mark.rate!r}\n")
        f.write("arrival_ms,task_id\n")
        for ev in trace.events:
            f.write(f"{ev.time_ms!r},{ev.task_id}\n")


def read_trace(path: str, n_tasks: Optional[int] = None) -> WorkloadTrace:
    """workload.py:270-321 (same validation and TraceParseError line numbers)."""
    events, marks = [], []
    seed, rng_algo, saw_header, last_time = 0, RNG_ALGO, False, -math.inf
    with open(path, "r", encoding="utf-8") as f:
        for lineno, raw in enumerate(f, start=1):
            line = raw.strip()
            if not line:
                continue
            if line.startswith("#"):
                parts = [p.strip() for p in line[1:].split(",")]
                try:
                    if parts[0] == "segment":
                        marks.append(SegmentMark(int(parts[1]), float(parts[2])))
                    elif parts[0] == "seed":
                        seed = int(parts[1])
                    elif parts[0] == "rng":
                        rng_algo = parts[1]
                except (IndexError, ValueError):
                    raise TraceParseError(f"malformed comment line: {line}", path, lineno)
                continue
            if not saw_header:
                if line != "arrival_ms,task_id":
                    raise TraceParseError(f"expected header 'arrival_ms,task_id', got {line!r}", path, lineno)
                saw_header = True
                continue
            cols = line.split(",")
            if len(cols) != 2:
                raise TraceParseError(f"expected 2 columns, got {len(cols)}", path, lineno)
            try:
                t, task = float(cols[0]), int(cols[1])
            except ValueError:
                raise TraceParseError(f"malformed row: {line}", path, lineno)
            if not math.isfinite(t) or t < 0:
                raise TraceParseError(f"arrival_ms must be finite and nonnegative: {cols[0]}", path, lineno)
            if t < last_time:
                raise TraceParseError("arrival times must be nondecreasing", path, lineno)
            if task < 0 or (n_tasks is not None and task >= n_tasks):
                raise TraceParseError(f"unknown task id {task}", path, lineno)
            last_time = t
            events.append(ArrivalEvent(t, task))
    if not saw_header:
        raise TraceParseError("missing header", path, 0)
    trace = WorkloadTrace(events=events, segment_marks=marks, seed=seed, rng_algo=rng_algo)
    trace.validate()
    return trace


def write_metrics_csv(run, path: str) -> None:
    """evalkit.py:300-305."""
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(METRICS_HEADER + "\n")
        for r in run.records:
            f.write(f"{r.index},{r.arrival_ms!r},{r.task_id},{r.tier_id},"
                    f"{r.reward!r},{r.realized_ms_per_token!r},{r.segment_rate!r}\n")


def read_metrics_csv(path: str):
    """evalkit.py:308-321."""
    from .evalkit import RequestRecord
    records = []
    with open(path, "r", encoding="utf-8") as f:
        header = f.readline().strip()
        if header != METRICS_HEADER:
            raise ValueError(f"{path}: unexpected metrics header {header!r}")
        for line in f:
            cols = line.strip().split(",")
            if len(cols) != 7:
                raise ValueError(f"{path}: expected 7 columns, got {len(cols)}")
            records.append(RequestRecord(int(cols[0]), float(cols[1]), int(cols[2]), int(cols[3]),
                                         float(cols[4]), float(cols[5]), float(cols[6])))
    return records


def summary_row(run, reward_spec) -> dict:
    """cli.py:145-160 (windowed + threshold_counts over the run's rewards)."""
    rewards = np.array([r.reward for r in run.records])
    w = _windowed(rewards)
    counts = {th: (int(np.sum(w == 1.0)) if th == 1.0 else int(np.sum(w >= th))) for th in THRESHOLDS}
    total_miss = float(np.mean([
        1.0 if r.realized_ms_per_token > reward_spec.tasks[r.task_id].deadline_ms_per_token else 0.0
        for r in run.records])) if run.records else math.nan
    row = {"n_requests": len(run.records),
           "mean_reward": float(rewards.mean()) if run.records else math.nan,
           "miss_fraction": total_miss,
           "mean_utility_per_gpu": float(rewards.mean() / run.gpu_count) if run.records else math.nan}
    for theta in THRESHOLDS:
        key = "windows_eq_%.2f" % theta if theta == 1.0 else "windows_ge_%.2f" % theta
        row[key] = counts[theta]
    return row


def write_summary(runs: Sequence, reward_spec, path: str) -> None:
    """cli.py:184-195."""
    rows = [summary_row(run, reward_spec) for run in runs]
    keys = list(rows[0].keys())
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write("trial," + ",".join(keys) + "\n")
        for k, row in enumerate(rows):
            f.write(f"{k}," + ",".join(repr(row[key]) if isinstance(row[key], float) else str(row[key])
                                       for key in keys) + "\n")


def write_per_rate(runs: Sequence, reward_spec, path: str) -> None:
    """cli.py:203-216."""
    by_rate, miss_by_rate = {}, {}
    for run in runs:
        for rec in run.records:
            by_rate.setdefault(rec.segment_rate, []).append(rec.reward)
            deadline = reward_spec.tasks[rec.task_id].deadline_ms_per_token
            miss_by_rate.setdefault(rec.segment_rate, []).append(
                1.0 if rec.realized_ms_per_token > deadline else 0.0)
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write("rate,mean_reward,miss_fraction,n_requests\n")
        for rate in sorted(by_rate):
            f.write(f"{rate!r},{float(np.mean(by_rate[rate]))!r},"
                    f"{float(np.mean(miss_by_rate[rate]))!r},{len(by_rate[rate])}\n")


def _windowed(v, window: int = 20) -> np.ndarray:
    """evalkit.py:217-226 (host; the device version is evalkit.windowed)."""
    v = np.asarray(v, dtype=float)
    if v.size < window:
        return np.empty(0)
    c = np.concatenate(([0.0], np.cumsum(v)))
    return (c[window:] - c[:-window]) / window
