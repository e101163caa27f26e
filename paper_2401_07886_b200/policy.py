"""Router on the GPU: encode / QNetwork.forward / select_action.

  encode           policy.py:52-65
  QNetwork.forward policy.py:111-118   -> be_qnet_route_f64 (fp64, warp per state)
  select_action    policy.py:125-132   -> same kernel, Philox epsilon draw
  route_tc         the batched router on the tensor cores (be_qnet_route_tc): same
                   actions, fp32 Q values
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .specs import QNetwork


class DeviceQNet:
    """fp64 QNetwork parameters resident on the GPU (BEQN1 layout)."""

    def __init__(self, net, device=None):
        dev = _lib.require_cuda(device)
        net = QNetwork.from_any(net)
        for a in (net.w1, net.b1, net.w2, net.b2):
            if not np.all(np.isfinite(a)):
                raise ValueError("non-finite network parameters")
        self.n_tasks, self.n_tiers, self.hidden = net.n_tasks, net.n_tiers, net.hidden
        self.w1 = torch.as_tensor(np.ascontiguousarray(net.w1), device=dev)
        self.b1 = torch.as_tensor(np.ascontiguousarray(net.b1), device=dev)
        self.w2 = torch.as_tensor(np.ascontiguousarray(net.w2), device=dev)
        self.b2 = torch.as_tensor(np.ascontiguousarray(net.b2), device=dev)

    @classmethod
    def of(cls, net, device=None) -> "DeviceQNet":
        return net if isinstance(net, cls) else cls(net, device)

    def weights(self) -> _lib.BeQWeights:
        w = _lib.BeQWeights()
        w.hidden = self.hidden
        w.n_tasks, w.n_tiers = self.n_tasks, self.n_tiers
        w.w1, w.b1, w.w2, w.b2 = (t.data_ptr() for t in (self.w1, self.b1, self.w2, self.b2))
        return w

    def to_host(self) -> QNetwork:
        return QNetwork(self.n_tasks, self.n_tiers, self.w1.cpu().numpy(), self.b1.cpu().numpy(),
                        self.w2.cpu().numpy(), self.b2.cpu().numpy())


def route(net, x: torch.Tensor, epsilon: float = 0.0, seed: int = 0, counter: int = 0,
          want_q: bool = True):
    """Batched select_action: x [B, D] fp64 on device -> (q [B, M], action u8 [B])."""
    dn = DeviceQNet.of(net)
    x = x.to(dtype=torch.float64).contiguous()
    if x.dim() != 2 or x.shape[1] != dn.n_tasks + dn.n_tiers + 1:
        raise ValueError(f"expected input dim {dn.n_tasks + dn.n_tiers + 1}")
    if not bool(torch.isfinite(x).all()):
        raise ValueError("non-finite network input")  # policy.py:115-116
    B = x.shape[0]
    q = torch.empty((B, dn.n_tiers), dtype=torch.float64, device=x.device) if want_q else None
    a = torch.empty(B, dtype=torch.uint8, device=x.device)
    w = dn.weights()
    L = _lib.load()
    _lib.check(L.be_qnet_route_f64(w, dn.n_tasks, dn.n_tiers, x.data_ptr(), B, float(epsilon),
                                   int(seed) & (2**64 - 1), int(counter) & (2**64 - 1),
                                   _lib.ptr(q), a.data_ptr(), _lib.stream_ptr()))
    return q, a


class TensorCoreRouter:
    """Batched select_action on the tensor cores (be_qnet_route_tc, route_tc.cu).

    Layer 1 runs as tcgen05 kind::tf32 MMAs (3xTF32 split, 256 states per tile,
    accumulators in TMEM); every greedy decision is certified by an error bound
    or re-evaluated with the fp64 router's exact arithmetic, so the actions
    equal `route()`'s; Q values are fp32 (within 1e-5 relative).  Owns the
    packed-weight workspace and a (states, fp64 re-evaluations) counter."""

    def __init__(self, net, device=None):
        self.net = DeviceQNet.of(net, device)
        dn = self.net
        L = _lib.load()
        if not L.be_qnet_route_tc_supported(dn.n_tasks, dn.n_tiers, dn.hidden):
            raise _lib.InvalidParameterError(
                "tensor-core router needs n_tiers <= 4, n_tasks + n_tiers + 2 <= 16, hidden % 32 == 0 <= 256")
        dev = dn.w1.device
        nbytes = int(L.be_qnet_route_tc_workspace_bytes(dn.hidden))
        self.workspace = torch.empty((nbytes + 15) // 16 * 4, dtype=torch.float32, device=dev)
        self.stats = torch.zeros(2, dtype=torch.int64, device=dev)

    def __call__(self, x: torch.Tensor, epsilon: float = 0.0, seed: int = 0, counter: int = 0,
                 want_q: bool = True, out: "torch.Tensor | None" = None, check: bool = True):
        dn = self.net
        x = x.to(dtype=torch.float64).contiguous()
        if x.dim() != 2 or x.shape[1] != dn.n_tasks + dn.n_tiers + 1:
            raise ValueError(f"expected input dim {dn.n_tasks + dn.n_tiers + 1}")
        if check and not bool(torch.isfinite(x).all()):
            raise ValueError("non-finite network input")  # policy.py:115-116
        B = x.shape[0]
        q = torch.empty((B, dn.n_tiers), dtype=torch.float32, device=x.device) if want_q else None
        a = out if out is not None else torch.empty(B, dtype=torch.uint8, device=x.device)
        w = dn.weights()
        L = _lib.load()
        _lib.check(L.be_qnet_route_tc(w, dn.n_tasks, dn.n_tiers, x.data_ptr(), B, float(epsilon),
                                      int(seed) & (2**64 - 1), int(counter) & (2**64 - 1), _lib.ptr(q),
                                      a.data_ptr(), self.workspace.data_ptr(), self.stats.data_ptr(),
                                      _lib.stream_ptr()))
        return q, a

    def fallback_stats(self, reset: bool = False) -> tuple:
        s = self.stats.tolist()
        if reset:
            self.stats.zero_()
        return int(s[0]), int(s[1])


def route_tc(net, x: torch.Tensor, epsilon: float = 0.0, seed: int = 0, counter: int = 0,
             want_q: bool = True):
    """Batched select_action on the tensor cores: (q fp32 [B, M], action u8 [B])."""
    return TensorCoreRouter(net, x.device)(x, epsilon, seed, counter, want_q)


def q_forward_batch(net, x) -> np.ndarray:
    """QNetwork.forward drop-in: numpy in, numpy out, computed on the GPU."""
    xa = np.asarray(x, dtype=np.float64)
    single = xa.ndim == 1
    dev = _lib.require_cuda()
    q, _ = route(net, torch.as_tensor(np.atleast_2d(xa), device=dev))
    out = q.cpu().numpy()
    return out[0] if single else out


def select_action(net, encoded, epsilon: float, rng) -> int:
    """select_action drop-in (policy.py:125-132); the exploration coin comes
    from the caller's numpy Generator exactly as in the reference, the greedy
    branch from the GPU forward."""
    if not 0.0 <= epsilon <= 1.0:
        raise ValueError("epsilon must lie in [0, 1]")
    n_tiers = QNetwork.from_any(net).n_tiers if not isinstance(net, DeviceQNet) else net.n_tiers
    if epsilon > 0.0 and rng.random() < epsilon:
        return int(rng.integers(0, n_tiers))
    return int(np.argmax(q_forward_batch(net, encoded)))


def encode(state, encoding) -> np.ndarray:
    """policy.py:52-65 (host helper for single states)."""
    if not 0 <= state.task_id < encoding.n_tasks:
        raise ValueError(f"task_id {state.task_id} out of range")
    if len(state.tier_batches) != encoding.n_tiers:
        raise ValueError("tier_batches length does not match encoding")
    if state.arrival_rate < 0:
        raise ValueError("arrival rate must be nonnegative")
    x = np.zeros(encoding.input_dim)
    x[state.task_id] = 1.0
    for m, b in enumerate(state.tier_batches):
        x[encoding.n_tasks + m] = b / encoding.batch_scales[m]
    x[-1] = state.arrival_rate / encoding.rate_scale
    return x
