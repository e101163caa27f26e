"""Shared test helpers: build specs from golden metadata, run the oracle."""
import numpy as np

import goldens
from oracle import oracle
from paper_2401_07886_b200 import specs


def tiers_of(meta):
    return [specs.ModelTierSpec(i, **t) for i, t in enumerate(meta["tiers"])]


def reward_of(meta):
    r = meta["reward"]
    return specs.RewardSpec(tasks=tuple(specs.TaskSpec(t["name"], t["deadline"], t["kind"])
                                        for t in r["tasks"]),
                            matrix=tuple(tuple(x) for x in r["matrix"]),
                            decay_per_ms=r["decay"], cutoff_fraction=r["cutoff"])


def enc_of(meta):
    return specs.StateEncoding(len(meta["reward"]["tasks"]), tuple(meta["enc"]["batch_scales"]),
                               meta["enc"]["rate_scale"])


def oracle_run(g, **kw):
    m = g["meta"]
    args = dict(tiers=m["tiers"], reward=m["reward"], arrival=g["arrival"], task=g["task"],
                seg_start=g["seg_start"], seg_rate=g["seg_rate"], net=goldens.net_for(m),
                static_tier=m["static_tier"], batch_scales=m["enc"]["batch_scales"],
                rate_scale=m["enc"]["rate_scale"], estimator_mode=m["estimator_mode"],
                reset=m["reset"])
    args.update(kw)
    return oracle.run_eval_oracle(**args)


def first_diff(a, b):
    d = np.nonzero(np.asarray(a) != np.asarray(b))[0]
    return int(d[0]) if d.size else -1


def _oracle_row(args):
    (kw, arrival, task, seg_start, seg_rate) = args
    from oracle import oracle as orc
    return orc.run_eval_oracle(arrival=arrival, task=task, seg_start=seg_start, seg_rate=seg_rate,
                               want_steps=False, **kw)


def oracle_rows(tb, rows, procs=None, **kw):
    """Run the oracle on env rows `rows` of a device TraceBatch (one host process
    per core).  kw: tiers, reward, net, batch_scales, rate_scale, estimator_mode,
    reset, static_tier.  Returns {row: oracle output dict}."""
    import multiprocessing as mp
    import os
    n_ev = None if tb.n_events is None else tb.n_events.cpu().numpy()
    offs = tb.seg_offsets.cpu().numpy()
    ss, sr = tb.seg_start.cpu().numpy(), tb.seg_rate.cpu().numpy()
    jobs = []
    for r in rows:
        n = tb.ld if n_ev is None else int(n_ev[r])
        jobs.append((kw, tb.arrival[r, :n].cpu().numpy(), tb.task[r, :n].cpu().numpy(),
                     ss[offs[r]:offs[r + 1]], sr[offs[r]:offs[r + 1]]))
    procs = max(1, min(procs or len(os.sched_getaffinity(0)), len(jobs)))
    with mp.get_context("spawn").Pool(procs) as pool:
        outs = pool.map(_oracle_row, jobs)
    return dict(zip(rows, outs))


def assert_rows_match_oracle(o, refs, deadlines, tasks_of_row):
    """Bit-exact: tier, miss flag and reward (and realized when recorded) of the
    GPU rollout outputs `o` against oracle outputs {row: dict}."""
    for r, ref in refs.items():
        n = ref["tier"].size
        flags = o.flags[r, :n].cpu().numpy()
        tier = flags & 0x3F
        assert np.array_equal(tier, ref["tier"]), f"env {r} tier first diff {first_diff(tier, ref['tier'])}"
        rw = o.reward[r, :n].cpu().numpy()
        assert np.array_equal(rw.view(np.int64), ref["reward"].view(np.int64)), \
            f"env {r} reward first diff {first_diff(rw, ref['reward'])}"
        miss = ((flags >> 7) & 1).astype(bool)
        ref_miss = ref["realized"] > np.asarray(deadlines)[tasks_of_row(r)[:n]]
        assert np.array_equal(miss, ref_miss), f"env {r} miss first diff {first_diff(miss, ref_miss)}"
        if o.realized is not None:
            rl = o.realized[r, :n].cpu().numpy()
            assert np.array_equal(rl.view(np.int64), ref["realized"].view(np.int64)), \
                f"env {r} realized first diff {first_diff(rl, ref['realized'])}"
