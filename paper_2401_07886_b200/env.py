"""Batched serving environment: E independent ClusterSims on one GPU.

  EnvBatch.reset  ClusterSim.__init__ / re-create (simcore.py:72-84, evalkit.py:189-191)
  EnvBatch.step   advance -> score -> estimator -> observe -> route -> submit
                  (evalkit.py:193-205, trainer.py:375-395; simcore.py:94-157)
  EnvBatch.drain  ClusterSim.drain (simcore.py:151-153)

Device state per env: one Rep header per replica (48 B) + a FIFO ring of
`ring_capacity` 16-byte slots per replica; see DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .policy import DeviceQNet


def _get(o, name, default=None):
    if isinstance(o, dict):
        return o.get(name, default)
    return getattr(o, name, default)


def make_cfg(tiers: Sequence, reward_spec, encoding=None, *, estimator_mode: str = "estimated",
             prior_rate: float = 1.0, reset_between_segments: bool = False,
             ring_capacity: int = 1024, skip_ahead: bool = True, q_screen: bool = True) -> _lib.BeCfg:
    """Pack ModelTierSpec / RewardSpec / StateEncoding / RateEstimator settings."""
    if estimator_mode not in ("estimated", "true-rate"):
        raise _lib.InvalidParameterError("mode must be one of ('estimated', 'true-rate')")
    if prior_rate <= 0:
        raise _lib.InvalidParameterError("prior_rate must be positive")
    tiers = list(tiers)
    M = len(tiers)
    if not tiers:
        raise _lib.InvalidParameterError("at least one tier required")
    if [int(_get(t, "tier_id", i)) for i, t in enumerate(tiers)] != list(range(M)):
        raise _lib.InvalidParameterError("tier_ids must be 0..M-1 in order")
    if M > _lib.MAX_TIERS:
        raise _lib.InvalidParameterError("at most 8 tiers")
    tasks = list(reward_spec.tasks)
    T = len(tasks)
    if T > _lib.MAX_TASKS:
        raise _lib.InvalidParameterError("at most 16 tasks")
    if len(reward_spec.matrix[0]) != M:
        raise ValueError("tier count must match reward matrix width")
    c = _lib.BeCfg()
    c.n_tiers, c.n_tasks = M, T
    for m, t in enumerate(tiers):
        c.tiers[m].replicas = int(t.replicas)
        c.tiers[m].max_batch = int(t.max_batch)
        c.tiers[m].tokens_per_request = int(_get(t, "tokens_per_request", 100))
        c.tiers[m].alpha_ms = float(t.alpha_ms)
        c.tiers[m].beta_ms = float(t.beta_ms)
    for k, task in enumerate(tasks):
        c.deadline[k] = float(task.deadline_ms_per_token)
        c.soft[k] = 1 if task.kind == "soft" else 0
        for m in range(M):
            c.matrix[k * M + m] = float(reward_spec.matrix[k][m])
    c.decay_per_ms = float(reward_spec.decay_per_ms)
    c.cutoff_fraction = float(reward_spec.cutoff_fraction)
    scales = (encoding.batch_scales if encoding is not None
              else [float(t.max_batch) for t in tiers])  # evalkit.py:164-166
    if len(scales) != M:
        raise ValueError("tier_batches length does not match encoding")
    for m in range(M):
        c.batch_scales[m] = float(scales[m])
    c.rate_scale = float(encoding.rate_scale) if encoding is not None else 48.0
    c.estimator_true_rate = 1 if estimator_mode == "true-rate" else 0
    c.reset_between_segments = 1 if reset_between_segments else 0
    c.prior_rate = float(prior_rate)
    c.ring_capacity = int(ring_capacity)
    c.skip_ahead = 1 if skip_ahead else 0
    c.q_screen = 1 if q_screen else 0
    return c


def default_ring_capacity(ld: int, n_envs: int, replicas: int, budget_bytes: int) -> int:
    """Smallest power of two that cannot overflow (> ld) when the budget allows,
    else the largest power of two within the budget (overflow is detected and
    reported, never silent)."""
    need = 1 << max(1, int(ld).bit_length())
    cap = need
    while cap > 64 and n_envs * replicas * cap * 16 > budget_bytes:
        cap //= 2
    return cap


class EnvBatch:
    """Owner of a be_env handle (E envs on one device)."""

    def __init__(self, tiers, reward_spec, n_envs: int, encoding=None, *,
                 estimator_mode: str = "estimated", prior_rate: float = 1.0,
                 reset_between_segments: bool = False, ring_capacity: int = 1024,
                 skip_ahead: bool = True, q_screen: bool = True, device=None):
        self.device = _lib.require_cuda(device)
        self.tiers = list(tiers)
        self.reward_spec = reward_spec
        self.encoding = encoding
        self.n_envs = int(n_envs)
        self.n_tiers = len(self.tiers)
        self.n_tasks = reward_spec.n_tasks if hasattr(reward_spec, "n_tasks") else len(reward_spec.tasks)
        self.cfg = make_cfg(tiers, reward_spec, encoding, estimator_mode=estimator_mode,
                            prior_rate=prior_rate, reset_between_segments=reset_between_segments,
                            ring_capacity=ring_capacity, skip_ahead=skip_ahead, q_screen=q_screen)
        self.ring_capacity = int(ring_capacity)
        self._L = _lib.load()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.be_env_create(ctypes.byref(self.cfg), self.n_envs,
                                             self.device.index or 0, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        return int(self._L.be_env_device_bytes(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.be_env_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, stream=None) -> None:
        _lib.check(self._L.be_env_check(self._h, _lib.stream_ptr(stream)))

    def screen_stats(self, reset: bool = False) -> tuple:
        """(screened decisions, fp64 fallbacks) of the greedy rollout's certified
        fp32 decision screen since the last reset (synchronises the device)."""
        out = (ctypes.c_int64 * 2)()
        _lib.check(self._L.be_env_screen_stats(self._h, out, 1 if reset else 0))
        return int(out[0]), int(out[1])

    def rollout_plan(self) -> dict:
        """What the last fused rollout on this handle launched (be_env_rollout_plan)."""
        out = (ctypes.c_int32 * 8)()
        _lib.check(self._L.be_env_rollout_plan(self._h, out))
        keys = ("n_tiers", "lanes_per_env", "true_rate", "throughput_variant", "skip_smem",
                "screen", "ctas_per_sm", "ctas")
        return dict(zip(keys, (int(x) for x in out)))

    def reset(self, mask: Optional[torch.Tensor] = None, stream=None) -> None:
        _lib.check(self._L.be_env_reset(self._h, _lib.ptr(mask), _lib.stream_ptr(stream)))

    def step(self, arrival: torch.Tensor, task: torch.Tensor, records: "StepRecords", *,
             true_rate: Optional[torch.Tensor] = None, policy=None, static_tier: int = -1,
             forced: Optional[torch.Tensor] = None, epsilon: float = 0.0, seed: int = 0,
             counter: int = 0, want_x: bool = False, stream=None) -> dict:
        """One routed request per env.  Returns device tensors obs [E, M] i32,
        rate [E] f64, action [E] u8, q [E, M] f64 and x [E, D] f64 (encoded state)."""
        E, M = self.n_envs, self.n_tiers
        dev = self.device
        _check_vec(arrival, "arrival", torch.float64, E, dev)
        _check_vec(task, "task", torch.uint8, E, dev)  # ids >= n_tasks: EINVAL from the kernel
        if true_rate is not None:
            _check_vec(true_rate, "true_rate", torch.float64, E, dev)
        if forced is not None:
            _check_vec(forced, "forced", torch.uint8, E, dev)
        out = dict(obs=torch.empty((E, M), dtype=torch.int32, device=dev),
                   rate=torch.empty(E, dtype=torch.float64, device=dev),
                   action=torch.empty(E, dtype=torch.uint8, device=dev))
        w = None
        if policy is not None and forced is None and static_tier < 0:
            dn = DeviceQNet.of(policy, dev)
            w = dn.weights()
            out["q"] = torch.empty((E, M), dtype=torch.float64, device=dev)
        if want_x:
            out["x"] = torch.empty((E, self.n_tasks + M + 1), dtype=torch.float64, device=dev)
        rec = records.struct()
        _lib.check(self._L.be_env_step(
            self._h, arrival.data_ptr(), task.data_ptr(), _lib.ptr(true_rate), _lib.ptr(forced),
            ctypes.byref(w) if w is not None else None, int(static_tier), float(epsilon),
            int(seed) & (2**64 - 1), int(counter) & (2**64 - 1), records.ld, ctypes.byref(rec),
            out["obs"].data_ptr(), out["rate"].data_ptr(), out["action"].data_ptr(),
            _lib.ptr(out.get("q")), _lib.ptr(out.get("x")), _lib.stream_ptr(stream)))
        return out

    def observe(self, arrival: torch.Tensor, task: torch.Tensor, records: "StepRecords", *,
                true_rate: Optional[torch.Tensor] = None, stream=None) -> dict:
        """First half of a step split around a router (be_env_step_observe): advance,
        score completions, estimator, observe, encode.  Returns x [E, D] f64,
        obs [E, M] i32, rate [E] f64 (device); no decision is made."""
        E, M, dev = self.n_envs, self.n_tiers, self.device
        _check_vec(arrival, "arrival", torch.float64, E, dev)
        _check_vec(task, "task", torch.uint8, E, dev)
        if true_rate is not None:
            _check_vec(true_rate, "true_rate", torch.float64, E, dev)
        out = dict(x=torch.empty((E, self.n_tasks + M + 1), dtype=torch.float64, device=dev),
                   obs=torch.empty((E, M), dtype=torch.int32, device=dev),
                   rate=torch.empty(E, dtype=torch.float64, device=dev))
        rec = records.struct()
        _lib.check(self._L.be_env_step_observe(
            self._h, arrival.data_ptr(), task.data_ptr(), _lib.ptr(true_rate), records.ld, ctypes.byref(rec),
            out["x"].data_ptr(), out["obs"].data_ptr(), out["rate"].data_ptr(), _lib.stream_ptr(stream)))
        return out

    def submit(self, arrival: torch.Tensor, task: torch.Tensor, action: torch.Tensor,
               records: "StepRecords", stream=None) -> None:
        """Second half (be_env_step_submit): submit every env's request to the tier
        in `action` (u8 [E], e.g. from TensorCoreRouter on observe()'s x)."""
        E, dev = self.n_envs, self.device
        _check_vec(arrival, "arrival", torch.float64, E, dev)
        _check_vec(task, "task", torch.uint8, E, dev)
        _check_vec(action, "action", torch.uint8, E, dev)
        rec = records.struct()
        _lib.check(self._L.be_env_step_submit(self._h, arrival.data_ptr(), task.data_ptr(), action.data_ptr(),
                                              records.ld, ctypes.byref(rec), _lib.stream_ptr(stream)))

    def drain(self, records: "StepRecords", stream=None) -> None:
        rec = records.struct()
        _lib.check(self._L.be_env_drain(self._h, records.ld, ctypes.byref(rec),
                                        _lib.stream_ptr(stream)))

    def new_segment(self, records: "StepRecords", mask: Optional[torch.Tensor] = None,
                    stream=None) -> None:
        """run_eval's stable-segment reset (evalkit.py:186-192) for the envs with
        mask[e] != 0 (all if None): drain into `records`, fresh replicas and an
        empty estimator window; request ids keep counting."""
        if mask is not None:
            _check_vec(mask, "mask", torch.uint8, self.n_envs, self.device)
        rec = records.struct()
        _lib.check(self._L.be_env_new_segment(self._h, _lib.ptr(mask), records.ld, ctypes.byref(rec),
                                              _lib.stream_ptr(stream)))


def _check_vec(t, name, dtype, n, dev):
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or t.device != dev or t.numel() < n \
            or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of >= {n} elements on {dev}")


class StepRecords:
    """Per-request outputs [E, ld] written at completion (indexed by request id
    modulo ld): flags = tier | miss << 7, reward f64, realized f64."""

    def __init__(self, n_envs: int, ld: int, device, want_realized: bool = True):
        self.ld = int(ld)
        self.flags = torch.zeros((n_envs, ld), dtype=torch.uint8, device=device)
        self.reward = torch.full((n_envs, ld), float("nan"), dtype=torch.float64, device=device)
        self.realized = (torch.full((n_envs, ld), float("nan"), dtype=torch.float64, device=device)
                         if want_realized else None)

    def struct(self) -> _lib.BeRecords:
        r = _lib.BeRecords()
        r.flags = self.flags.data_ptr()
        r.reward = self.reward.data_ptr()
        r.realized = _lib.ptr(self.realized)
        return r
