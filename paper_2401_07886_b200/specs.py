"""Host-side mirror of the reference's value types.

Same names, fields, defaults and validation errors as the reference
(`besteffort` 0.1.0) so callers can swap packages; every function in this
package also accepts the reference's own objects (duck-typed by attribute).

  ModelTierSpec            simcore.py:21-37
  TaskSpec, RewardSpec     reward.py:32-91
  StateEncoding            policy.py:23-42
  ArrivalEvent, SegmentMark, WorkloadTrace   workload.py:39-91
  QNetwork (parameters), BEQN1 checkpoints   policy.py:68-118, :193-232
  DEFAULT_CONFIG cluster / rewards           config.py:25-85
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import numpy as np

from ._lib import InvalidParameterError

HARD, SOFT = "hard", "soft"
RNG_ALGO = "pcg64"
CHECKPOINT_MAGIC = "BEQN1"
HIDDEN_DEFAULT = 256

DEFAULT_TASKS = (("hellaswag", 40.0, HARD), ("copa", 40.0, HARD), ("piqa", 40.0, HARD),
                 ("openbookqa", 40.0, HARD))
DEFAULT_MATRIX = ((0.45, 0.78, 1.00), (0.80, 0.95, 1.00), (0.82, 0.96, 1.00),
                  (0.70, 0.94, 1.00))
# config.py:31-36 — the authoritative cluster calibration
DEFAULT_TIERS = (
    dict(name="small", replicas=4, alpha_ms=4.75, beta_ms=0.25, max_batch=128,
         tokens_per_request=100, baseline_max_batch=160),
    dict(name="medium", replicas=4, alpha_ms=8.0, beta_ms=1.2, max_batch=32,
         tokens_per_request=100, baseline_max_batch=48),
    dict(name="large", replicas=4, alpha_ms=28.0, beta_ms=4.0, max_batch=8,
         tokens_per_request=100, baseline_max_batch=12),
)


class CheckpointError(ValueError):
    pass


@dataclass(frozen=True)
class ModelTierSpec:
    tier_id: int
    replicas: int
    alpha_ms: float
    beta_ms: float
    max_batch: int
    tokens_per_request: int = 100
    name: str = ""

    def __post_init__(self):
        if self.replicas < 1:
            raise InvalidParameterError("replicas must be >= 1")
        if self.alpha_ms <= 0 or self.beta_ms < 0:
            raise InvalidParameterError("alpha_ms must be > 0 and beta_ms >= 0")
        if self.max_batch < 1 or self.tokens_per_request < 1:
            raise InvalidParameterError("max_batch and tokens_per_request must be >= 1")


def default_tiers(baseline: bool = False, replicas: Optional[int] = None) -> list[ModelTierSpec]:
    """AppConfig.tiers() of the shipped config (config.py:128-139)."""
    out = []
    for i, t in enumerate(DEFAULT_TIERS):
        out.append(ModelTierSpec(i, replicas or t["replicas"], t["alpha_ms"], t["beta_ms"],
                                 t["baseline_max_batch"] if baseline else t["max_batch"],
                                 t["tokens_per_request"], t["name"]))
    return out


@dataclass(frozen=True)
class TaskSpec:
    name: str
    deadline_ms_per_token: float
    kind: str = HARD

    def __post_init__(self):
        if self.deadline_ms_per_token <= 0:
            raise ValueError(f"task {self.name}: deadline must be positive")
        if self.kind not in (HARD, SOFT):
            raise ValueError(f"task {self.name}: kind must be '{HARD}' or '{SOFT}'")


@dataclass(frozen=True)
class RewardSpec:
    tasks: tuple
    matrix: tuple
    decay_per_ms: float = 0.01
    cutoff_fraction: float = 0.10

    def __post_init__(self):
        if not self.tasks or not self.matrix:
            raise ValueError("tasks and matrix must be nonempty")
        if len(self.matrix) != len(self.tasks):
            raise ValueError("matrix must have one row per task")
        width = len(self.matrix[0])
        if any(len(row) != width for row in self.matrix):
            raise ValueError("matrix rows must have equal length")
        if any(v < 0 or v > 1 for row in self.matrix for v in row):
            raise ValueError("matrix entries must lie in [0, 1]")
        if not 0 < self.decay_per_ms <= 1 or not 0 < self.cutoff_fraction <= 1:
            raise ValueError("decay_per_ms and cutoff_fraction must lie in (0, 1]")

    @property
    def n_tasks(self) -> int:
        return len(self.tasks)

    @property
    def n_tiers(self) -> int:
        return len(self.matrix[0])

    def with_kind(self, kind: str) -> "RewardSpec":
        return replace(self, tasks=tuple(replace(t, kind=kind) for t in self.tasks))

    def with_deadlines(self, deadlines: dict) -> "RewardSpec":
        return replace(self, tasks=tuple(
            replace(t, deadline_ms_per_token=deadlines.get(t.name, t.deadline_ms_per_token))
            for t in self.tasks))

    @classmethod
    def default(cls) -> "RewardSpec":
        return cls(tasks=tuple(TaskSpec(*t) for t in DEFAULT_TASKS), matrix=DEFAULT_MATRIX)


@dataclass(frozen=True)
class StateEncoding:
    n_tasks: int
    batch_scales: tuple
    rate_scale: float = 48.0

    def __post_init__(self):
        if self.n_tasks < 1 or not self.batch_scales:
            raise ValueError("n_tasks and batch_scales must be nonempty")
        if self.rate_scale <= 0 or any(s <= 0 for s in self.batch_scales):
            raise ValueError("scales must be positive")

    @property
    def n_tiers(self) -> int:
        return len(self.batch_scales)

    @property
    def input_dim(self) -> int:
        return self.n_tasks + self.n_tiers + 1


@dataclass(frozen=True)
class ArrivalEvent:
    time_ms: float
    task_id: int


@dataclass(frozen=True)
class SegmentMark:
    start_index: int
    rate: float


@dataclass
class WorkloadTrace:
    events: list
    segment_marks: list
    seed: int
    rng_algo: str = RNG_ALGO

    def __len__(self) -> int:
        return len(self.events)

    def validate(self) -> None:
        last = -math.inf
        for i, ev in enumerate(self.events):
            if ev.time_ms < 0 or ev.time_ms < last:
                raise ValueError(f"event {i}: times must be nonnegative and sorted")
            last = ev.time_ms
        if self.segment_marks:
            if self.segment_marks[0].start_index != 0:
                raise ValueError("first segment mark must start at index 0")
            starts = [m.start_index for m in self.segment_marks]
            if any(b < a for a, b in zip(starts, starts[1:])):
                raise ValueError("segment mark start indices must be nondecreasing")

    def event_rates(self) -> np.ndarray:
        return event_rates(self)

    def segments(self) -> list:
        out = []
        starts = [m.start_index for m in self.segment_marks]
        for k, mark in enumerate(self.segment_marks):
            end = starts[k + 1] if k + 1 < len(starts) else len(self.events)
            if end > mark.start_index:
                out.append((mark.start_index, end, mark.rate))
        return out


def event_rates(trace) -> np.ndarray:
    """WorkloadTrace.event_rates (workload.py:74-81) for any trace-like object.
    Indices not covered by a mark are NaN (the reference leaves them
    uninitialised)."""
    n = len(trace.events)
    rates = np.full(n, np.nan)
    marks = list(trace.segment_marks)
    starts = [m.start_index for m in marks]
    for k, mark in enumerate(marks):
        end = starts[k + 1] if k + 1 < len(starts) else n
        rates[mark.start_index:end] = mark.rate
    return rates


def param_layout(n_tasks: int, n_tiers: int, hidden: int) -> tuple:
    """(name, shape, offset) of w1, b1, w2, b2 in the flat fp64 parameter vector —
    the BEQN1 payload order and the device learner's `params` layout."""
    d = n_tasks + n_tiers + 1
    out, off = [], 0
    for name, shape in (("w1", (d, hidden)), ("b1", (hidden,)), ("w2", (hidden, n_tiers)),
                        ("b2", (n_tiers,))):
        out.append((name, shape, off))
        off += int(np.prod(shape))
    return tuple(out)


def _param_property(name: str):
    def get(self):
        return self._views[name]

    def put(self, value):
        v = self._views[name]
        value = np.asarray(value, dtype=np.float64)
        if value.shape != v.shape:
            raise ValueError(f"{name}: expected shape {v.shape}, got {value.shape}")
        v[...] = value

    return property(get, put, doc=f"{name} (a view into `flat`)")


class QNetwork:
    """Router MLP parameters (the reference QNetwork, policy.py:68-118), held as ONE
    contiguous fp64 vector `flat` in BEQN1 payload order (w1 | b1 | w2 | b2);
    w1/b1/w2/b2 are views into it.  The GPU path uploads `flat` in one copy and
    checkpoints are `flat` behind a two-line header.  `forward` runs on the GPU."""

    w1 = _param_property("w1")
    b1 = _param_property("b1")
    w2 = _param_property("w2")
    b2 = _param_property("b2")

    def __init__(self, n_tasks, n_tiers, w1, b1, w2, b2):
        t, m = int(n_tasks), int(n_tiers)
        arrays = [np.asarray(x) for x in (w1, b1, w2, b2)]
        h = arrays[0].shape[1] if arrays[0].ndim == 2 else -1
        layout = param_layout(t, m, max(h, 0))
        for k, ((name, shape, _), arr) in enumerate(zip(layout, arrays)):
            if arr.shape != shape or h < 0:
                raise ValueError("layer 1 shape mismatch" if k < 2 else "layer 2 shape mismatch")
        self._init_flat(t, m, h, np.concatenate([x.astype(np.float64).ravel() for x in arrays]))

    def _init_flat(self, t: int, m: int, h: int, flat: np.ndarray) -> None:
        self.n_tasks, self.n_tiers, self.hidden = t, m, h
        self.input_dim = t + m + 1
        self.flat = flat
        self._views = {name: flat[off:off + int(np.prod(shape))].reshape(shape)
                       for name, shape, off in param_layout(t, m, h)}

    @classmethod
    def from_flat(cls, n_tasks: int, n_tiers: int, hidden: int, flat) -> "QNetwork":
        flat = np.array(flat, dtype=np.float64).ravel()
        need = param_layout(n_tasks, n_tiers, hidden)[-1]
        if flat.size != need[2] + n_tiers:
            raise ValueError(f"expected {need[2] + n_tiers} parameters, got {flat.size}")
        net = cls.__new__(cls)
        net._init_flat(int(n_tasks), int(n_tiers), int(hidden), flat)
        return net

    @classmethod
    def init_random(cls, n_tasks, n_tiers, hidden=HIDDEN_DEFAULT, rng=None):
        """Reference initialisation (policy.py:86-98): w1 ~ U(+-sqrt(6/D)), then
        w2 ~ U(+-sqrt(6/H)) from the same Generator (same draws, same order),
        zero biases."""
        g = np.random.default_rng() if rng is None else rng
        net = cls.from_flat(n_tasks, n_tiers, hidden,
                            np.zeros(param_layout(n_tasks, n_tiers, hidden)[-1][2] + n_tiers))
        lim_in = math.sqrt(6.0 / net.input_dim)
        net.w1 = g.uniform(-lim_in, lim_in, size=net.w1.shape)
        lim_h = math.sqrt(6.0 / hidden)
        net.w2 = g.uniform(-lim_h, lim_h, size=net.w2.shape)
        return net

    @classmethod
    def from_any(cls, net) -> "QNetwork":
        if isinstance(net, cls):
            return net
        if isinstance(net, dict):
            m = len(net["b2"])
            return cls(np.shape(net["w1"])[0] - m - 1, m, net["w1"], net["b1"], net["w2"], net["b2"])
        return cls(net.n_tasks, net.n_tiers, net.w1, net.b1, net.w2, net.b2)

    def params(self):
        return [self.w1, self.b1, self.w2, self.b2]

    def copy(self) -> "QNetwork":
        return QNetwork.from_flat(self.n_tasks, self.n_tiers, self.hidden, self.flat.copy())

    def load_from(self, other) -> None:
        src = other.flat if isinstance(other, QNetwork) else np.concatenate(
            [np.asarray(x, np.float64).ravel() for x in (other.w1, other.b1, other.w2, other.b2)])
        if src.shape != self.flat.shape:
            raise ValueError("parameter count mismatch")
        self.flat[...] = src

    def forward(self, x):
        from .policy import q_forward_batch
        return q_forward_batch(self, x)


# ---------------------------------------------------------------- BEQN1 checkpoints
# File = b"BEQN1\n" + b"<n_tasks> <n_tiers> <hidden>\n" + the flat parameter vector as
# little-endian float64 (policy.py:193-199 format).  Read errors are CheckpointError
# with the reference's messages (policy.py:202-232).

def save_checkpoint(net, path: str) -> None:
    q = QNetwork.from_any(net)
    head = f"{CHECKPOINT_MAGIC}\n{q.n_tasks} {q.n_tiers} {q.hidden}\n".encode("ascii")
    with open(path, "wb") as f:
        f.write(head + q.flat.astype("<f8").tobytes())


def _take_line(blob: bytes, pos: int) -> tuple:
    """The line starting at `pos` including its newline (file.readline semantics)."""
    end = blob.find(b"\n", pos)
    end = len(blob) if end < 0 else end + 1
    return blob[pos:end], end


def load_checkpoint(path: str, n_tasks=None, n_tiers=None) -> QNetwork:
    with open(path, "rb") as f:
        blob = f.read()
    line, pos = _take_line(blob, 0)
    magic = line.decode("ascii", errors="replace").strip()
    if magic != CHECKPOINT_MAGIC:
        raise CheckpointError(f"{path}: bad magic {magic!r}")
    line, pos = _take_line(blob, pos)
    fields = line.decode("ascii", errors="replace").split()
    try:
        if len(fields) != 3:
            raise ValueError
        dims = [int(v) for v in fields]
    except ValueError:
        raise CheckpointError(f"{path}: malformed dimension header")
    t, m, h = dims
    if min(dims) < 1:
        raise CheckpointError(f"{path}: nonpositive dimensions")
    if (n_tasks is not None and t != n_tasks) or (n_tiers is not None and m != n_tiers):
        raise CheckpointError(f"{path}: dimensions ({t}, {m}) do not match expected "
                              f"({n_tasks}, {n_tiers})")
    count = param_layout(t, m, h)[-1][2] + m
    payload = memoryview(blob)[pos:]
    if len(payload) < 8 * count:
        raise CheckpointError(f"{path}: truncated parameter payload")
    if len(payload) > 8 * count:
        raise CheckpointError(f"{path}: trailing bytes after parameters")
    return QNetwork.from_flat(t, m, h, np.frombuffer(payload, dtype="<f8"))
