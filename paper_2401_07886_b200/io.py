"""Reference-format CSV files for batched GPU results, host side.

The reference writes its files one Python record at a time (trace files
workload.py:258-267, per-request metrics evalkit.py:300-305, the CLI's summary
and per-rate tables cli.py:145-216).  Here every file is a *column table*:
numpy columns (straight from a rollout's device outputs, or from EvalRun
records) are formatted column-wise — float64 columns with numpy's shortest
round-trip formatting, which is exactly Python's `repr(float)` — and joined
into the file in one write.  The bytes equal the reference's for the same
values (tests/test_io_cpu.py pins sha256 digests of reference-written files).

Readers parse whole files: lines are classified first (blank / comment /
header / row), row columns are converted in bulk, and the validation runs
vectorised; the error raised is the one the reference's line-by-line reader
raises first — same exception type, message and line number
(workload.py:270-321, evalkit.py:308-321).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from ._lib import InvalidParameterError
from .specs import RNG_ALGO, ArrivalEvent, SegmentMark, WorkloadTrace

METRICS_COLUMNS = ("request_index", "arrival_ms", "task_id", "tier_id", "reward",
                   "realized_ms_per_token", "segment_rate")
METRICS_HEADER = ",".join(METRICS_COLUMNS)
TRACE_HEADER = "arrival_ms,task_id"
PER_RATE_COLUMNS = ("rate", "mean_reward", "miss_fraction", "n_requests")
THRESHOLDS = (1.00, 0.99, 0.98, 0.96, 0.94)  # cli.py summary columns (config.THRESHOLDS)


class TraceParseError(InvalidParameterError):
    """workload.py:32-36: a malformed trace file, with path and line number."""

    def __init__(self, message: str, path: str, lineno: int):
        super().__init__(f"{path}:{lineno}: {message}")
        self.path = path
        self.lineno = lineno


# ------------------------------------------------------------------ formatting
def _fmt(col) -> np.ndarray:
    """One column as strings: float64 -> shortest repr (== repr(float)), ints -> str."""
    a = np.asarray(col)
    if a.dtype.kind == "f":
        return a.astype(np.float64).astype(str)
    if a.dtype.kind in "iub":
        return a.astype(np.int64).astype(str)
    return a.astype(str)


def _table(columns: Sequence, header: Optional[str] = None, preamble: Sequence[str] = ()) -> str:
    """Join formatted columns into CSV text ('\\n' line ends, trailing newline)."""
    cols = [_fmt(c) for c in columns]
    n = len(cols[0]) if cols else 0
    out = list(preamble)
    if header is not None:
        out.append(header)
    if n:
        rows = cols[0]
        for c in cols[1:]:
            rows = np.char.add(np.char.add(rows, ","), c)
        out.extend(rows.tolist())
    return "".join(line + "\n" for line in out)


def _write(path: str, text: str) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(text)


# ------------------------------------------------------------------ trace files
def write_trace(trace, path: str) -> None:
    """Trace file (workload.py:258-267 format): `# rng`, `# seed` and one `# segment`
    comment per mark, then `arrival_ms,task_id` rows."""
    if hasattr(trace, "validate"):
        trace.validate()
    pre = [f"# rng,{getattr(trace, 'rng_algo', RNG_ALGO)}", f"# seed,{trace.seed}"]
    marks = list(trace.segment_marks)
    if marks:
        seg = _table([np.array([m.start_index for m in marks], np.int64),
                      np.array([m.rate for m in marks], np.float64)])
        pre += ["# segment," + s for s in seg.splitlines()]
    t = np.fromiter((e.time_ms for e in trace.events), np.float64, len(trace.events))
    k = np.fromiter((e.task_id for e in trace.events), np.int64, len(trace.events))
    _write(path, _table([t, k], TRACE_HEADER, pre))


def write_trace_arrays(arrival, task, seg_start, seg_rate, seed: int, path: str,
                       rng_algo: str = RNG_ALGO) -> None:
    """The same file straight from arrays (e.g. one row of a device TraceBatch)."""
    a = np.asarray(arrival, np.float64)
    if a.size and (not np.all(np.isfinite(a)) or a[0] < 0 or np.any(np.diff(a) < 0)):
        raise InvalidParameterError("arrival times must be finite, nonnegative and sorted")
    pre = [f"# rng,{rng_algo}", f"# seed,{seed}"]
    if len(seg_start):
        pre += ["# segment," + s for s in
                _table([np.asarray(seg_start, np.int64), np.asarray(seg_rate, np.float64)]).splitlines()]
    _write(path, _table([a, np.asarray(task, np.int64)], TRACE_HEADER, pre))


def _text_lines(path: str):
    """(lineno, stripped text) of the non-blank lines, numbered like iterating the
    file object (universal newlines, '\n'-separated)."""
    with open(path, "r", encoding="utf-8") as f:
        raw = f.read().split("\n")
    return [(i + 1, s.strip()) for i, s in enumerate(raw) if s.strip()]


def _comment(text: str):
    """Parse a `# key,value...` line: ('segment', SegmentMark) | ('seed', int) |
    ('rng', str) | (None, None) for unknown keys.  Raises IndexError/ValueError."""
    fields = [x.strip() for x in text[1:].split(",")]
    key = fields[0]
    if key == "segment":
        return key, SegmentMark(int(fields[1]), float(fields[2]))
    if key == "seed":
        return key, int(fields[1])
    if key == "rng":
        return key, fields[1]
    return None, None


def read_trace(path: str, n_tasks: Optional[int] = None) -> WorkloadTrace:
    """Validating trace reader (workload.py:270-321 semantics and errors).

    One pass classifies the lines and stops at the first *structural* error
    (malformed comment, wrong header, wrong column count, unparsable number);
    the data rows before it are then validated in bulk.  A row failure earlier
    in the file wins over the structural error, as in a line-by-line reader."""
    marks, meta = [], {"seed": 0, "rng": RNG_ALGO}
    header_seen = False
    rows_at, times, tasks, raw_t = [], [], [], []
    pending = None  # (lineno, message) of the first structural error
    for lineno, text in _text_lines(path):
        if text.startswith("#"):
            try:
                key, val = _comment(text)
            except (IndexError, ValueError):
                pending = (lineno, f"malformed comment line: {text}")
                break
            if key == "segment":
                marks.append(val)
            elif key is not None:
                meta[key] = val
            continue
        if not header_seen:
            if text != TRACE_HEADER:
                pending = (lineno, f"expected header '{TRACE_HEADER}', got {text!r}")
                break
            header_seen = True
            continue
        cols = text.split(",")
        if len(cols) != 2:
            pending = (lineno, f"expected 2 columns, got {len(cols)}")
            break
        try:
            t, k = float(cols[0]), int(cols[1])
        except ValueError:
            pending = (lineno, f"malformed row: {text}")
            break
        rows_at.append(lineno)
        times.append(t)
        tasks.append(k)
        raw_t.append(cols[0])
    # task ids stay Python ints (object array): any size parses, as in the reference
    _check_trace_rows(np.array(times, np.float64), np.array(tasks, dtype=object), rows_at, raw_t,
                      path, n_tasks)
    if pending is not None:
        raise TraceParseError(pending[1], path, pending[0])
    if not header_seen:
        raise TraceParseError("missing header", path, 0)
    events = [ArrivalEvent(t, k) for t, k in zip(times, tasks)]
    trace = WorkloadTrace(events=events, segment_marks=marks, seed=meta["seed"], rng_algo=meta["rng"])
    trace.validate()
    return trace


def _check_trace_rows(times, tasks, linenos, raw_t, path, n_tasks):
    """Vectorised row checks; raises for the first offending row, with the
    reference's per-row check order (finite and nonnegative time, nondecreasing
    order, task id range)."""
    if times.size == 0:
        return
    bad_time = ~np.isfinite(times) | (times < 0)
    # every row before the first failure was accepted, so the time a row must
    # not precede is the running maximum of the accepted times before it
    ok_t = np.where(bad_time, -math.inf, times)
    prev = np.concatenate(([-math.inf], np.maximum.accumulate(ok_t)[:-1]))
    bad_order = ~bad_time & (times < prev)
    bad_task = (tasks < 0).astype(bool)
    if n_tasks is not None:
        bad_task |= (tasks >= n_tasks).astype(bool)
    fail = bad_time | bad_order | bad_task
    if not fail.any():
        return
    j = int(np.argmax(fail))
    if bad_time[j]:
        raise TraceParseError(f"arrival_ms must be finite and nonnegative: {raw_t[j]}", path, linenos[j])
    if bad_order[j]:
        raise TraceParseError("arrival times must be nondecreasing", path, linenos[j])
    raise TraceParseError(f"unknown task id {int(tasks[j])}", path, linenos[j])


# ------------------------------------------------------------------ metrics
def _record_columns(run) -> list:
    recs = run.records
    n = len(recs)

    def col(attr, dt):
        return np.fromiter((getattr(r, attr) for r in recs), dt, n)

    return [col("index", np.int64), col("arrival_ms", np.float64), col("task_id", np.int64),
            col("tier_id", np.int64), col("reward", np.float64),
            col("realized_ms_per_token", np.float64), col("segment_rate", np.float64)]


def write_metrics_csv(run, path: str) -> None:
    """Per-request metrics CSV (evalkit.py:300-305 format) of an EvalRun."""
    _write(path, _table(_record_columns(run), METRICS_HEADER))


def write_metrics_arrays(path: str, arrival, task, tier, reward, realized, segment_rate) -> None:
    """The same file straight from one env's rollout arrays (e.g. a row of
    RolloutOutputs.tier / reward / realized and TraceBatch.event_rates)."""
    n = len(arrival)
    _write(path, _table([np.arange(n, dtype=np.int64), arrival, task, tier, reward, realized,
                         segment_rate], METRICS_HEADER))


def read_metrics_csv(path: str):
    """evalkit.py:308-321 semantics: header check, 7 columns per row."""
    from .evalkit import RequestRecord
    with open(path, "r", encoding="utf-8") as f:
        lines = f.read().split("\n")
    first = lines[0].strip() if lines else ""
    if first != METRICS_HEADER:
        raise ValueError(f"{path}: unexpected metrics header {first!r}")
    body = lines[1:]
    if body and body[-1] == "":
        body = body[:-1]  # the file's final newline
    split = [s.strip().split(",") for s in body]
    for cols in split:
        if len(cols) != len(METRICS_COLUMNS):
            raise ValueError(f"{path}: expected 7 columns, got {len(cols)}")
    conv = (int, float, int, int, float, float, float)
    return [RequestRecord(*(c(v) for c, v in zip(conv, cols))) for cols in split]


# ------------------------------------------------------------------ CLI tables
def _windows(rewards: np.ndarray, window: int = 20) -> np.ndarray:
    """Trailing means (evalkit.py:217-226): sequential fp64 prefix sum differences."""
    if rewards.size < window:
        return np.empty(0)
    c = np.empty(rewards.size + 1)
    c[0] = 0.0
    np.cumsum(rewards, out=c[1:])
    return (c[window:] - c[:-window]) / window


def _miss(run, reward_spec) -> np.ndarray:
    dl = np.array([t.deadline_ms_per_token for t in reward_spec.tasks])
    cols = _record_columns(run)
    return (cols[5] > dl[cols[2]]).astype(np.float64)


def summary_row(run, reward_spec) -> dict:
    """One row of the CLI summary table (cli.py:145-160 columns)."""
    cols = _record_columns(run)
    rewards = cols[4]
    w = _windows(rewards)
    n = rewards.size
    out = {"n_requests": n,
           "mean_reward": float(rewards.mean()) if n else math.nan,
           "miss_fraction": float(np.mean(_miss(run, reward_spec))) if n else math.nan,
           "mean_utility_per_gpu": float(rewards.mean() / run.gpu_count) if n else math.nan}
    for th in THRESHOLDS:
        if th == 1.0:
            out["windows_eq_1.00"] = int(np.count_nonzero(w == 1.0))
        else:
            out[f"windows_ge_{th:.2f}"] = int(np.count_nonzero(w >= th))
    return out


def write_summary(runs: Sequence, reward_spec, path: str) -> None:
    """Summary CSV (cli.py:184-195 format): `trial` then the summary_row columns."""
    rows = [summary_row(r, reward_spec) for r in runs]
    keys = list(rows[0])
    columns = [np.arange(len(rows), dtype=np.int64)]
    for k in keys:
        vals = [row[k] for row in rows]
        columns.append(np.array(vals, np.float64 if isinstance(vals[0], float) else np.int64))
    _write(path, _table(columns, "trial," + ",".join(keys)))


def write_per_rate(runs: Sequence, reward_spec, path: str) -> None:
    """Per-rate CSV (cli.py:203-216 format): mean reward, miss fraction and count
    per segment rate, ascending; means over the requests in run/record order."""
    rate = np.concatenate([_record_columns(r)[6] for r in runs])
    rew = np.concatenate([_record_columns(r)[4] for r in runs])
    miss = np.concatenate([_miss(r, reward_spec) for r in runs])
    keys = np.unique(rate[~np.isnan(rate)]) if rate.size else np.empty(0)
    if np.isnan(rate).any():
        raise ValueError("records without a segment rate")
    means, misses, counts = [], [], []
    for v in keys:
        sel = rate == v
        means.append(float(np.mean(rew[sel])))
        misses.append(float(np.mean(miss[sel])))
        counts.append(int(sel.sum()))
    _write(path, _table([keys, np.array(means), np.array(misses), np.array(counts, np.int64)],
                        ",".join(PER_RATE_COLUMNS)))
