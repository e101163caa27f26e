"""ctypes binding of the C ABI in include/be200.h (libbe200.so, built in-tree).

There is no CPU fallback: if the shared library is missing or CUDA is not
available every entry point raises.  Arguments are raw device pointers taken
from torch tensors (torch is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BE200_LIB: alternative build of the same library (A/B experiments on the GPU box)
LIB_PATH = os.environ.get("BE200_LIB") or os.path.join(_HERE, "libbe200.so")

BE_OK, BE_EINVAL, BE_ECAPACITY, BE_ECUDA, BE_ENONFINITE = range(5)
MAX_TIERS, MAX_TASKS, MAX_LANES = 8, 16, 32


class InvalidParameterError(ValueError):
    """Mirror of besteffort.workload.InvalidParameterError (workload.py:28-29)."""


class CapacityError(RuntimeError):
    """A replica FIFO ring overflowed: the env must be recreated larger."""


class CudaError(RuntimeError):
    pass


class BeTier(ctypes.Structure):
    _fields_ = [("replicas", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("tokens_per_request", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("alpha_ms", ctypes.c_double), ("beta_ms", ctypes.c_double)]


class BeCfg(ctypes.Structure):
    _fields_ = [("n_tiers", ctypes.c_int32), ("n_tasks", ctypes.c_int32),
                ("tiers", BeTier * MAX_TIERS),
                ("deadline", ctypes.c_double * MAX_TASKS),
                ("soft", ctypes.c_int32 * MAX_TASKS),
                ("matrix", ctypes.c_double * (MAX_TASKS * MAX_TIERS)),
                ("decay_per_ms", ctypes.c_double), ("cutoff_fraction", ctypes.c_double),
                ("batch_scales", ctypes.c_double * MAX_TIERS), ("rate_scale", ctypes.c_double),
                ("estimator_true_rate", ctypes.c_int32), ("reset_between_segments", ctypes.c_int32),
                ("prior_rate", ctypes.c_double), ("ring_capacity", ctypes.c_int32),
                ("skip_ahead", ctypes.c_int32), ("q_screen", ctypes.c_int32),
                ("_pad2", ctypes.c_int32)]


class BeTraceSoa(ctypes.Structure):
    _fields_ = [("n_envs", ctypes.c_int32), ("_pad", ctypes.c_int32), ("ld", ctypes.c_int64),
                ("arrival_ms", ctypes.c_void_p), ("task", ctypes.c_void_p),
                ("n_events", ctypes.c_void_p), ("seg_offsets", ctypes.c_void_p),
                ("seg_start", ctypes.c_void_p), ("seg_rate", ctypes.c_void_p),
                ("seg_bucket", ctypes.c_void_p), ("env_ready", ctypes.c_void_p),
                ("envs_per_ready", ctypes.c_int32), ("ready_value", ctypes.c_int32)]


class BeQWeights(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("n_tasks", ctypes.c_int16), ("n_tiers", ctypes.c_int16),
                ("w1", ctypes.c_void_p), ("b1", ctypes.c_void_p),
                ("w2", ctypes.c_void_p), ("b2", ctypes.c_void_p)]


MAX_THETA = 8


class BeThresholds(ctypes.Structure):  # passed by value
    _fields_ = [("n", ctypes.c_int32), ("_pad", ctypes.c_int32), ("theta", ctypes.c_double * MAX_THETA)]


class BeRecords(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_void_p), ("reward", ctypes.c_void_p),
                ("realized", ctypes.c_void_p), ("obs", ctypes.c_void_p),
                ("rate", ctypes.c_void_p), ("q", ctypes.c_void_p)]


class BeGenCfg(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_tasks", ctypes.c_int32), ("n_task_ids", ctypes.c_int32),
                ("task_ids", ctypes.c_int32 * MAX_TASKS), ("n_rates", ctypes.c_int32),
                ("truncate", ctypes.c_int32), ("rate_ld", ctypes.c_int64), ("rates", ctypes.c_void_p),
                ("hold_ms", ctypes.c_double), ("n", ctypes.c_int64), ("seg_capacity", ctypes.c_int64)]


GEN_STABLE, GEN_UNPRED_TIME, GEN_UNPRED_REQ = 0, 1, 2


class BeLearnerCfg(ctypes.Structure):
    _fields_ = [("n_tasks", ctypes.c_int32), ("n_tiers", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("n_envs", ctypes.c_int32), ("replay_capacity", ctypes.c_int64),
                ("pending_capacity", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("warmup", ctypes.c_int64), ("target_sync_every", ctypes.c_int64),
                ("discount", ctypes.c_double), ("learning_rate", ctypes.c_double),
                ("adam", ctypes.c_int32), ("huber", ctypes.c_int32),
                ("rate_low", ctypes.c_double), ("rate_high", ctypes.c_double),
                ("regime_equal_time", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("regime_mean_seconds", ctypes.c_double), ("regime_mean_requests", ctypes.c_double)]


class BeTrainIterCfg(ctypes.Structure):
    _fields_ = [("workload_seed", ctypes.c_uint64), ("policy_seed", ctypes.c_uint64),
                ("sample_seed", ctypes.c_uint64), ("epsilon_start", ctypes.c_double),
                ("epsilon_end", ctypes.c_double), ("epsilon_decay_steps", ctypes.c_int64),
                ("updates_per_step", ctypes.c_int32), ("phase", ctypes.c_int32),
                ("update_index", ctypes.c_int32), ("use_gate", ctypes.c_int32),
                ("router", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class BeLearnerViews(ctypes.Structure):
    _fields_ = [("online", BeQWeights), ("target", BeQWeights), ("params", ctypes.c_void_p),
                ("grad", ctypes.c_void_p), ("nparam", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("loss", ctypes.c_void_p), ("counters", ctypes.c_void_p),
                ("ring_states", ctypes.c_void_p), ("ring_next_states", ctypes.c_void_p),
                ("ring_actions", ctypes.c_void_p), ("ring_rewards", ctypes.c_void_p),
                ("ring_cont", ctypes.c_void_p), ("ring_state", ctypes.c_void_p),
                ("pending_x", ctypes.c_void_p), ("pending_action", ctypes.c_void_p),
                ("pending_flags", ctypes.c_void_p), ("pending_reward", ctypes.c_void_p),
                ("workload_state", ctypes.c_void_p), ("gate", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I32, _I64, _U64, _D, _SZ = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t

# name -> (restype, argtypes); the exported surface of include/be200.h
SIGNATURES = {
    "be_last_error": (ctypes.c_char_p, []),
    "be_abi_version": (_I32, []),
    "be_env_create": (_I32, [ctypes.POINTER(BeCfg), _I32, _I32, ctypes.POINTER(_P)]),
    "be_env_destroy": (_I32, [_P]),
    "be_env_device_bytes": (_SZ, [_P]),
    "be_env_reset": (_I32, [_P, _P, _P]),
    "be_env_check": (_I32, [_P, _P]),
    "be_env_status_async": (_I32, [_P, _P, _P]),
    "be_env_screen_stats": (_I32, [_P, _P, _I32]),
    "be_env_rollout_plan": (_I32, [_P, _P]),
    "be_env_step": (_I32, [_P, _P, _P, _P, _P, ctypes.POINTER(BeQWeights), _I32, _D, _U64, _U64,
                           _I64, ctypes.POINTER(BeRecords), _P, _P, _P, _P, _P, _P]),
    "be_env_drain": (_I32, [_P, _I64, ctypes.POINTER(BeRecords), _P]),
    "be_env_new_segment": (_I32, [_P, _P, _I64, ctypes.POINTER(BeRecords), _P]),
    "be_env_step_observe": (_I32, [_P, _P, _P, _P, _I64, ctypes.POINTER(BeRecords), _P, _P, _P, _P]),
    "be_env_step_submit": (_I32, [_P, _P, _P, _P, _I64, ctypes.POINTER(BeRecords), _P]),
    "be_rollout_greedy": (_I32, [_P, ctypes.POINTER(BeTraceSoa), ctypes.POINTER(BeQWeights), _I32,
                                 _P, ctypes.POINTER(BeRecords), _P]),
    "be_qnet_route_f64": (_I32, [ctypes.POINTER(BeQWeights), _I32, _I32, _P, _I32, _D, _U64, _U64,
                                 _P, _P, _P]),
    "be_qnet_route_tc_supported": (_I32, [_I32, _I32, _I32]),
    "be_qnet_route_tc_workspace_bytes": (_SZ, [_I32]),
    "be_qnet_route_tc": (_I32, [ctypes.POINTER(BeQWeights), _I32, _I32, _P, _I32, _D, _U64, _U64,
                                _P, _P, _P, _P, _P]),
    "be_reduce_eval": (_I32, [ctypes.POINTER(BeTraceSoa), _P, _P, _I32, BeThresholds, _I32, _P, _P, _P,
                              _P, _P, _P]),
    "be_reduce_selection": (_I32, [ctypes.POINTER(BeTraceSoa), _P, _I32, _I32, _I32, _P, _P]),
    "be_windowed": (_I32, [ctypes.POINTER(BeTraceSoa), _P, _I32, _P, _P]),
    "be_trace_gen_stable": (_I32, [_I32, _I64, _I64, _I64, _P, _I32, _U64, _P, _P, _P]),
    "be_trace_gen": (_I32, [ctypes.POINTER(BeGenCfg), _I32, _I64, _I64, _U64, _P, _P, _P, _P, _P, _P,
                            _P, _P]),
    "be_learner_create": (_I32, [ctypes.POINTER(BeLearnerCfg), _I32, ctypes.POINTER(_P)]),
    "be_learner_destroy": (_I32, [_P]),
    "be_learner_set_params": (_I32, [_P, _P, _P, _P, _P, _P]),
    "be_learner_views": (_I32, [_P, ctypes.POINTER(BeLearnerViews)]),
    "be_learner_workload": (_I32, [_P, _U64, _I64, _P, _P, _P, _P]),
    "be_learner_commit": (_I32, [_P, _I64, _P]),
    "be_learner_backward": (_I32, [_P, _U64, _U64, _P, _P]),
    "be_learner_backward_batch": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _P]),
    "be_learner_apply": (_I32, [_P, _I32, _P]),
    "be_learner_check": (_I32, [_P, _P]),
    "be_train_iteration": (_I32, [_P, _P, ctypes.POINTER(BeTrainIterCfg), _P]),
    "be_learner_exchange_buffer": (_I32, [_P, ctypes.POINTER(_P), ctypes.POINTER(_SZ)]),
    "be_learner_ipc_handle": (_I32, [_P, _P]),
    "be_learner_set_peers": (_I32, [_P, _I32, _I32, _P]),
    "be_learner_open_peers_ipc": (_I32, [_P, _I32, _I32, _P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libbe200.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (or make -C paper_2401_07886_b200/csrc)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == BE_OK:
        return
    msg = load().be_last_error().decode(errors="replace")
    if rc == BE_EINVAL:
        raise InvalidParameterError(msg)
    if rc == BE_ECAPACITY:
        raise CapacityError(msg)
    if rc == BE_ENONFINITE:
        raise ValueError(msg)
    raise CudaError(msg)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2401_07886_b200 needs a CUDA device (sm_100a); no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if d.type != "cuda":
        raise RuntimeError(f"paper_2401_07886_b200 runs on CUDA devices only, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
