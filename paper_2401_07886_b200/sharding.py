"""Multi-GPU plumbing: environment sharding and the end-of-run statistics reduce.

Environments never interact (evalkit.py:154-209 keeps no cross-instance
state), so rollouts shard by global env id with no data-path collective; the
only exchanges are:
  * the int64 evaluation statistics, summed once at the end (exact);
  * the per-rank f64 reward sums, gathered and added in rank order so the
    result is identical for every launch with the same world size;
  * max-over-ranks of the step time (timing only).
Works with the "nccl" backend on GPUs and "gloo" on CPU (tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous env slice [lo, hi) of rank `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dev(device):
    if device is not None:
        return device
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")


def max_over_ranks(x: float, device=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_stats(red, device=None) -> dict:
    """All-reduce a ReduceResult's per-env statistics into whole-job totals
    (same keys as ReduceResult.totals())."""
    dev = _dev(device)
    ints = torch.cat([red.win_counts.sum(0), red.n_windows.sum().reshape(1),
                      red.bucket_miss.sum(0), red.bucket_req.sum(0)]).to(dev, torch.int64)
    dist.all_reduce(ints, op=dist.ReduceOp.SUM)
    n_theta, K = red.win_counts.shape[1], red.bucket_miss.shape[1]
    # f64 reward sums: per-rank sum (fixed order), gathered, added in rank order
    local = red.bucket_reward.to(dev, torch.float64).sum(0)
    world = dist.get_world_size()
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    rws = np.zeros(K)
    for p in parts:
        rws = rws + p.cpu().numpy()
    v = ints.cpu().numpy()
    wc, nw = v[:n_theta], int(v[n_theta])
    miss, req = v[n_theta + 1:n_theta + 1 + K], v[n_theta + 1 + K:]
    return dict(thresholds=list(red.thresholds), win_counts=wc.tolist(), n_windows=nw,
                window_fraction=(wc / max(nw, 1)).tolist(), requests=req.tolist(),
                misses=miss.tolist(), availability=(1.0 - miss / np.maximum(req, 1)).tolist(),
                mean_reward=(rws / np.maximum(req, 1)).tolist())


def broadcast_params(tensors, src: int = 0) -> None:
    """Replicate Q-network parameters from `src` (12.3 KB at fp32, 24.6 KB fp64)."""
    for t in tensors:
        dist.broadcast(t, src)


def allreduce_mean_(grad: torch.Tensor) -> torch.Tensor:
    """Data-parallel learner: sum gradients over ranks, then scale by 1/world."""
    dist.all_reduce(grad, op=dist.ReduceOp.SUM)
    grad.mul_(1.0 / dist.get_world_size())
    return grad
