"""Fixture generator: learner I/O recorded from the UNMODIFIED reference trainer.

Test infrastructure only (SURVEY.md §8c goldens, item 4).  Fills the reference
`ReplayBuffer` (pkg/src/besteffort/trainer.py:101-163) with transitions of a
reference rollout (the committed `run_unpredictable-1_trained.npz`: s_i, a_i,
r_i, s_{i+1}, cont = 1, encoded as policy.py:52-65) and runs the reference
`train_step` (trainer.py:276-290 -> _StepKernel.compute :238-264 -> Adam/SGD
:177-208 -> target sync :288-289) for a few steps per (loss, optimizer) case,
recording for every step the sampled indices (the same `rng.integers` draw
`ReplayBuffer.sample` makes, trainer.py:158-163), the loss, the gradients and the
online/target parameters after the step.

Output: tests/golden/learner_<loss>_<opt>.npz.  Usage (build container):
    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_learner_golden.py
"""
import copy
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))

from besteffort.policy import QNetwork, load_checkpoint  # noqa: E402
from besteffort.trainer import (ReplayBuffer, TrainConfig, _StepKernel, make_optimizer,  # noqa: E402
                                train_step)

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [("huber", "adam"), ("squared", "adam"), ("huber", "sgd")]
STEPS = 6
BATCH = 512
LR = 1e-3
SYNC = 2


def transitions():
    z = np.load(os.path.join(HERE, "run_unpredictable-1_trained.npz"))
    meta = json.loads(str(z["meta"]))
    T = len(meta["reward"]["tasks"])
    scales = np.array(meta["enc"]["batch_scales"])
    n = len(z["arrival"])
    x = np.zeros((n, T + 3 + 1))
    x[np.arange(n), z["task"]] = 1.0
    x[:, T:T + 3] = z["obs"] / scales
    x[:, -1] = z["rate"] / meta["enc"]["rate_scale"]
    return x[:-1], z["tier"][:-1].astype(np.intp), z["reward"][:-1], x[1:], np.ones(n - 1)


def main():
    s, a, r, s2, c = transitions()
    base = load_checkpoint(os.path.join(HERE, "trained_seed7.beqn"))
    for loss, opt in CASES:
        cfg = TrainConfig(batch_size=BATCH, buffer_capacity=len(a), learning_rate=LR, loss=loss,
                          optimizer=opt, target_sync_every=SYNC, warmup=0)
        buf = ReplayBuffer(len(a), s.shape[1])
        for i in range(len(a)):
            buf.push(s[i], int(a[i]), float(r[i]), s2[i], 1.0)
        online = QNetwork(base.n_tasks, base.n_tiers, base.w1.copy(), base.b1.copy(),
                          base.w2.copy(), base.b2.copy())
        target = QNetwork(base.n_tasks, base.n_tiers, base.w1.copy(), base.b1.copy(),
                          base.w2.copy(), base.b2.copy())
        optimizer = make_optimizer(cfg, online.params())
        kernel = _StepKernel(s.shape[1], online.hidden, online.n_tiers, BATCH)
        rng = np.random.default_rng(11)
        rec = {k: [] for k in ("idx", "loss", "grad", "params", "target")}
        for step in range(1, STEPS + 1):
            idx = copy.deepcopy(rng).integers(0, buf.size, size=BATCH)
            lv = train_step(online, target, buf, cfg, step, optimizer, rng, kernel)
            rec["idx"].append(idx)
            rec["loss"].append(lv)
            rec["grad"].append(np.concatenate([g.ravel() for g in kernel.grads()]))
            rec["params"].append(np.concatenate([p.ravel() for p in online.params()]))
            rec["target"].append(np.concatenate([p.ravel() for p in target.params()]))
        meta = dict(loss=loss, optimizer=opt, batch=BATCH, lr=LR, target_sync_every=SYNC,
                    discount=cfg.discount, steps=STEPS, numpy=np.__version__,
                    source="besteffort.trainer.train_step (reference), rng default_rng(11)")
        out = os.path.join(HERE, f"learner_{loss}_{opt}.npz")
        np.savez_compressed(out, meta=json.dumps(meta), **{k: np.array(v) for k, v in rec.items()})
        print("wrote", out, "loss", rec["loss"])


if __name__ == "__main__":
    main()
