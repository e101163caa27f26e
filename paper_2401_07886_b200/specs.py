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


class QNetwork:
    """QNetwork parameters (policy.py:68-118), fp64 host arrays.

    `forward` runs on the GPU (route kernel); there is no CPU forward."""

    def __init__(self, n_tasks, n_tiers, w1, b1, w2, b2):
        self.n_tasks = int(n_tasks)
        self.n_tiers = int(n_tiers)
        self.hidden = int(np.shape(w1)[1])
        self.input_dim = self.n_tasks + self.n_tiers + 1
        if np.shape(w1) != (self.input_dim, self.hidden) or np.shape(b1) != (self.hidden,):
            raise ValueError("layer 1 shape mismatch")
        if np.shape(w2) != (self.hidden, self.n_tiers) or np.shape(b2) != (self.n_tiers,):
            raise ValueError("layer 2 shape mismatch")
        self.w1 = np.asarray(w1, dtype=np.float64)
        self.b1 = np.asarray(b1, dtype=np.float64)
        self.w2 = np.asarray(w2, dtype=np.float64)
        self.b2 = np.asarray(b2, dtype=np.float64)

    @classmethod
    def init_random(cls, n_tasks, n_tiers, hidden=HIDDEN_DEFAULT, rng=None):
        """policy.py:86-98: U(+-sqrt(6/fan_in)) weights, zero biases."""
        rng = rng if rng is not None else np.random.default_rng()
        d = n_tasks + n_tiers + 1
        b1, b2 = math.sqrt(6.0 / d), math.sqrt(6.0 / hidden)
        return cls(n_tasks, n_tiers, w1=rng.uniform(-b1, b1, size=(d, hidden)),
                   b1=np.zeros(hidden), w2=rng.uniform(-b2, b2, size=(hidden, n_tiers)),
                   b2=np.zeros(n_tiers))

    @classmethod
    def from_any(cls, net) -> "QNetwork":
        if isinstance(net, cls):
            return net
        if isinstance(net, dict):
            w1 = np.asarray(net["w1"])
            return cls(w1.shape[0] - len(net["b2"]) - 1, len(net["b2"]), net["w1"], net["b1"],
                       net["w2"], net["b2"])
        return cls(net.n_tasks, net.n_tiers, net.w1, net.b1, net.w2, net.b2)

    def params(self):
        return [self.w1, self.b1, self.w2, self.b2]

    def copy(self) -> "QNetwork":
        return QNetwork(self.n_tasks, self.n_tiers, self.w1.copy(), self.b1.copy(),
                        self.w2.copy(), self.b2.copy())

    def load_from(self, other) -> None:
        for dst, src in zip(self.params(), (other.w1, other.b1, other.w2, other.b2)):
            np.copyto(dst, src)

    def forward(self, x):
        from .policy import q_forward_batch
        return q_forward_batch(self, x)


def save_checkpoint(net, path: str) -> None:
    """policy.py:193-199: magic line, dims line, fp64 LE W1, b1, W2, b2."""
    with open(path, "wb") as f:
        f.write(f"{CHECKPOINT_MAGIC}\n".encode("ascii"))
        f.write(f"{net.n_tasks} {net.n_tiers} {np.shape(net.w1)[1]}\n".encode("ascii"))
        for p in (net.w1, net.b1, net.w2, net.b2):
            f.write(np.ascontiguousarray(p, dtype="<f8").tobytes())


def load_checkpoint(path: str, n_tasks=None, n_tiers=None) -> QNetwork:
    """policy.py:202-232 (same errors)."""
    with open(path, "rb") as f:
        magic = f.readline().decode("ascii", errors="replace").strip()
        if magic != CHECKPOINT_MAGIC:
            raise CheckpointError(f"{path}: bad magic {magic!r}")
        header = f.readline().decode("ascii", errors="replace").split()
        if len(header) != 3:
            raise CheckpointError(f"{path}: malformed dimension header")
        try:
            t, m, hidden = (int(v) for v in header)
        except ValueError:
            raise CheckpointError(f"{path}: malformed dimension header")
        if t < 1 or m < 1 or hidden < 1:
            raise CheckpointError(f"{path}: nonpositive dimensions")
        if (n_tasks is not None and t != n_tasks) or (n_tiers is not None and m != n_tiers):
            raise CheckpointError(f"{path}: dimensions ({t}, {m}) do not match expected "
                                  f"({n_tasks}, {n_tiers})")
        d = t + m + 1
        arrays = []
        for shape in [(d, hidden), (hidden,), (hidden, m), (m,)]:
            count = int(np.prod(shape))
            buf = f.read(count * 8)
            if len(buf) != count * 8:
                raise CheckpointError(f"{path}: truncated parameter payload")
            arrays.append(np.frombuffer(buf, dtype="<f8").reshape(shape).copy())
        if f.read(1):
            raise CheckpointError(f"{path}: trailing bytes after parameters")
    return QNetwork(t, m, *arrays)
