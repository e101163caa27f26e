"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's hot path used as the checker for the CUDA
path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
may import this module; the product package never does.

* `run_eval_oracle` wraps the plain-C rollout restatement (env_oracle.c,
  which cites pkg/src/besteffort/{evalkit,simcore,workload,reward,policy}.py
  line by line).
* `windowed`, `threshold_counts` restate pkg/src/besteffort/evalkit.py:217-241
  (sequential fp64 prefix sum, then (c[k+w]-c[k])/w; theta == 1.0 counts exact
  peaks only).
* `miss_fractions_by_rate` restates evalkit.py:61-68.
* `learner_step` restates the Double-Q / Huber / Adam update:
  trainer.py:166-174 (td_targets_double_q), :211-267 (_StepKernel),
  :177-199 (Adam), :276-290 (train_step), policy.py:146-190 (q_gradient).

Parity pins: tests/test_oracle_golden.py checks every function here against
fixtures produced by the reference itself (tests/golden/make_golden.py) and
against the reference's own known-answer tests.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _Tier(ctypes.Structure):
    _fields_ = [("replicas", ctypes.c_int), ("alpha", ctypes.c_double),
                ("beta", ctypes.c_double), ("max_batch", ctypes.c_int),
                ("tokens", ctypes.c_int)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "build", "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "build", "liboracle.so")
        if not os.path.exists(path):
            path = build()
        _LIB = ctypes.CDLL(path)
        _LIB.oracle_run_eval.restype = ctypes.c_int
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _get(o, *names, default=None):
    for n in names:
        if isinstance(o, dict) and n in o:
            return o[n]
        if hasattr(o, n):
            return getattr(o, n)
    return default


def run_eval_oracle(*, tiers, reward, arrival, task, seg_start, seg_rate, net=None,
                    static_tier=-1, forced_actions=None, batch_scales=None, rate_scale=48.0,
                    estimator_mode="estimated", prior_rate=1.0, reset=False,
                    want_steps=True):
    """Greedy rollout of one env.  `tiers`: sequence of objects/dicts with
    replicas, alpha_ms, beta_ms, max_batch, tokens_per_request.  `reward`:
    dict(tasks=[{deadline, kind}], matrix, decay, cutoff) or a RewardSpec."""
    M = len(tiers)
    tarr = (_Tier * M)()
    for m, t in enumerate(tiers):
        tarr[m].replicas = int(_get(t, "replicas"))
        tarr[m].alpha = float(_get(t, "alpha_ms"))
        tarr[m].beta = float(_get(t, "beta_ms"))
        tarr[m].max_batch = int(_get(t, "max_batch"))
        tarr[m].tokens = int(_get(t, "tokens_per_request", default=100))
    if isinstance(reward, dict):
        deadline = np.array([t["deadline"] for t in reward["tasks"]], np.float64)
        soft = np.array([t["kind"] == "soft" for t in reward["tasks"]], np.int32)
        matrix = np.ascontiguousarray(np.array(reward["matrix"], np.float64))
        decay, cutoff = float(reward["decay"]), float(reward["cutoff"])
    else:
        deadline = np.array([t.deadline_ms_per_token for t in reward.tasks], np.float64)
        soft = np.array([t.kind == "soft" for t in reward.tasks], np.int32)
        matrix = np.ascontiguousarray(np.array(reward.matrix, np.float64))
        decay, cutoff = float(reward.decay_per_ms), float(reward.cutoff_fraction)
    T = deadline.size
    arrival = np.ascontiguousarray(arrival, np.float64)
    task = np.ascontiguousarray(task, np.uint8)
    N = arrival.size
    seg_start = np.ascontiguousarray(seg_start, np.int64)
    seg_rate = np.ascontiguousarray(seg_rate, np.float64)
    if batch_scales is None:
        batch_scales = [float(_get(t, "max_batch")) for t in tiers]
    scales = np.ascontiguousarray(batch_scales, np.float64)
    if net is not None:
        w1 = np.ascontiguousarray(_get(net, "w1"), np.float64)
        b1 = np.ascontiguousarray(_get(net, "b1"), np.float64)
        w2 = np.ascontiguousarray(_get(net, "w2"), np.float64)
        b2 = np.ascontiguousarray(_get(net, "b2"), np.float64)
        hidden = w1.shape[1]
    else:
        w1 = b1 = w2 = b2 = None
        hidden = 0
        if static_tier < 0 and forced_actions is None:
            raise ValueError("need a net, a static tier or forced actions")
    fa = None if forced_actions is None else np.ascontiguousarray(forced_actions, np.uint8)
    tier = np.zeros(N, np.uint8)
    rw = np.zeros(N)
    rl = np.zeros(N)
    obs = np.zeros((N, M), np.int32) if want_steps else None
    rate = np.zeros(N) if want_steps else None
    q = np.full((N, M), np.nan) if (want_steps and net is not None) else None
    L = lib()
    rc = L.oracle_run_eval(
        ctypes.c_int(M), tarr, ctypes.c_int(T), _p(deadline), _p(soft), _p(matrix),
        ctypes.c_double(decay), ctypes.c_double(cutoff), _p(scales), ctypes.c_double(rate_scale),
        _p(w1), _p(b1), _p(w2), _p(b2), ctypes.c_int(hidden), ctypes.c_int(static_tier),
        _p(fa), ctypes.c_int64(N), _p(arrival), _p(task), ctypes.c_int64(seg_start.size),
        _p(seg_start), _p(seg_rate), ctypes.c_int(1 if estimator_mode == "true-rate" else 0),
        ctypes.c_double(prior_rate), ctypes.c_int(1 if reset else 0), _p(tier), _p(rw), _p(rl),
        _p(obs), _p(rate), _p(q))
    if rc != 0:
        raise ValueError("oracle_run_eval: invalid input")
    return dict(tier=tier, reward=rw, realized=rl, obs=obs, rate=rate, q=q)


# ---------------------------------------------------------------- reducers
def windowed(values, window=20):
    """evalkit.py:217-226 — c = [0, cumsum(v)] (sequential fp64), (c[w:]-c[:-w])/w."""
    v = np.asarray(values, dtype=float)
    if v.size < window:
        return np.empty(0)
    c = np.concatenate(([0.0], np.cumsum(v)))
    return (c[window:] - c[:-window]) / window


def threshold_counts(w, thresholds):
    """evalkit.py:229-241 — theta == 1.0 counts exact peak windows only."""
    w = np.asarray(w, dtype=float)
    return [int(np.sum(w == 1.0)) if th == 1.0 else int(np.sum(w >= th)) for th in thresholds]


def miss_fractions_by_rate(realized, task, event_rates, deadlines):
    """evalkit.py:61-68 — strict `realized > deadline[task]`, grouped by segment rate."""
    out = {}
    dl = np.asarray(deadlines)[np.asarray(task, int)]
    miss = np.asarray(realized) > dl
    for rate in np.unique(event_rates):
        sel = event_rates == rate
        out[float(rate)] = float(np.mean(miss[sel]))
    return out


# ---------------------------------------------------------------- learner
def forward(w1, b1, w2, b2, x):
    h = np.maximum(x @ w1 + b1, 0.0)
    return h, h @ w2 + b2


def learner_step(params, target, batch, *, discount, adam_state, lr, loss="huber",
                 beta1=0.9, beta2=0.999, eps=1e-8):
    """One train_step update in fp64 (trainer.py:238-267, :190-199).

    params/target: dict w1,b1,w2,b2 (fp64).  batch: states [B,D], actions [B],
    rewards [B], next_states [B,D], cont [B].  adam_state: dict t, m{...}, v{...}
    (mutated).  Returns (loss, grads, new_params)."""
    s, a, r, s2, c = batch
    a = np.asarray(a, np.intp)
    n = s.shape[0]
    rows = np.arange(n)
    _, q2 = forward(params["w1"], params["b1"], params["w2"], params["b2"], s2)
    best = q2.argmax(axis=1)
    _, q2t = forward(target["w1"], target["b1"], target["w2"], target["b2"], s2)
    y = r + c * discount * q2t[rows, best]
    h, q = forward(params["w1"], params["b1"], params["w2"], params["b2"], s)
    res = q[rows, a] - y
    if loss == "huber":
        ab = np.abs(res)
        loss_val = float(np.mean(np.where(ab <= 1.0, 0.5 * res ** 2, ab - 0.5)))
        dq = np.clip(res, -1.0, 1.0) / n
    else:
        loss_val = float(np.mean(0.5 * res ** 2))
        dq = res / n
    g = np.zeros_like(q)
    g[rows, a] = dq
    grads = dict(w2=h.T @ g, b2=g.sum(axis=0))
    dh = g @ params["w2"].T
    dh[h <= 0.0] = 0.0
    grads["w1"] = s.T @ dh
    grads["b1"] = dh.sum(axis=0)
    adam_state["t"] += 1
    t = adam_state["t"]
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    new = {}
    for k in ("w1", "b1", "w2", "b2"):
        m = adam_state["m"][k] = adam_state["m"][k] * beta1 + (1.0 - beta1) * grads[k]
        v = adam_state["v"][k] = adam_state["v"][k] * beta2 + (1.0 - beta2) * grads[k] * grads[k]
        new[k] = params[k] - lr * (m / bc1) / (np.sqrt(v / bc2) + eps)
    return loss_val, grads, new


def adam_init(params):
    return dict(t=0, m={k: np.zeros_like(v) for k, v in params.items()},
                v={k: np.zeros_like(v) for k, v in params.items()})
