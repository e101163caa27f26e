"""B200-native (sm_100a) hot path of *Learned Best-Effort LLM Serving* (arXiv 2401.07886).

Drop-in GPU implementations of the reference package's (`besteffort`)
environment step, router and evaluation interfaces, batched over thousands of
independent environments.  All compute runs in hand-written CUDA kernels
(libbe200.so, C ABI in include/be200.h); there is no CPU fallback.
"""
from ._lib import CapacityError, CudaError, InvalidParameterError  # noqa: F401
from .specs import (ArrivalEvent, CheckpointError, ModelTierSpec, QNetwork, RewardSpec,  # noqa: F401
                    SegmentMark, StateEncoding, TaskSpec, WorkloadTrace, default_tiers,
                    load_checkpoint, save_checkpoint)
from .trace import TraceBatch  # noqa: F401
from .env import EnvBatch, StepRecords, make_cfg  # noqa: F401
from .policy import DeviceQNet, TensorCoreRouter, route, route_tc, select_action  # noqa: F401
from .evalkit import (EvalRun, GreedyRollout, RequestRecord, ReduceResult, reduce_eval,  # noqa: F401
                      run_eval, run_eval_batch, THRESHOLDS, WINDOW)

__version__ = "0.1.0"
