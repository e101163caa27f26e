"""Differential tests of the host I/O against the reference's own functions
(run where the reference is importable: /root/reference/pkg/src in the build
container, or the baseline/_ref install; skipped elsewhere).

  * read_trace on randomly corrupted trace files: same accept/raise decision,
    same exception message (path:lineno: text) — workload.py:270-321;
  * write_trace / write_metrics_csv / summary / per-rate writers: same bytes on
    random records — workload.py:258-267, evalkit.py:300-305, cli.py:145-216;
  * BEQN1: same bytes written, same CheckpointError message on corrupted files,
    same parameters read — policy.py:193-232;
  * QNetwork.init_random: same draws from the same Generator — policy.py:86-98."""
import os
import sys

import numpy as np
import pytest

from paper_2401_07886_b200 import io as beio
from paper_2401_07886_b200 import specs
from paper_2401_07886_b200.evalkit import EvalRun, RequestRecord

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = ["/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")]


def _ref():
    for p in _CANDIDATES:
        if os.path.isdir(os.path.join(p, "besteffort")):
            if p not in sys.path:
                sys.path.append(p)
            import besteffort  # noqa: F401
            return True
    return False


pytestmark = pytest.mark.skipif(not _ref(), reason="reference package not importable here")


def _random_trace_text(rng):
    lines = []
    if rng.random() < 0.8:
        lines.append("# rng,pcg64")
    if rng.random() < 0.8:
        lines.append(f"# seed,{int(rng.integers(0, 1000))}")
    t = 0.0
    n = int(rng.integers(0, 12))
    body = []
    for i in range(n):
        t += float(rng.exponential(50.0))
        body.append(f"{t!r},{int(rng.integers(0, 4))}")
    lines.append("arrival_ms,task_id")
    lines += body
    if rng.random() < 0.5:
        lines.insert(min(2, len(lines)), f"# segment,0,{float(rng.uniform(0.5, 20))!r}")
    # corruptions, each with some probability
    mut = [
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "1.0"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "# segment,x,2"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "# seed,abc"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "nan,1"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "-3.0,1"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "0.5,0"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "1e9,9"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "abc,1"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), ""),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "   "),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "time,task"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "# foo,1"),
        lambda L: L.remove("arrival_ms,task_id"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "5.0,-1"),
        lambda L: L.insert(int(rng.integers(0, len(L) + 1)), "inf,0"),
    ]
    for f in mut:
        if rng.random() < 0.12:
            f(lines)
    return "\n".join(lines) + ("\n" if rng.random() < 0.9 else "")


def _outcome(fn, path, n_tasks):
    try:
        tr = fn(path, n_tasks=n_tasks)
        return ("ok", [(e.time_ms, e.task_id) for e in tr.events],
                [(m.start_index, m.rate) for m in tr.segment_marks], tr.seed, tr.rng_algo)
    except Exception as e:  # noqa: BLE001 — the type and message are what we compare
        return ("err", type(e).__name__, str(e))


def test_read_trace_matches_reference_on_corrupted_files(tmp_path):
    from besteffort.workload import read_trace as ref_read
    rng = np.random.default_rng(2024)
    path = str(tmp_path / "t.csv")
    n_err = 0
    for _ in range(600):
        with open(path, "w") as f:
            f.write(_random_trace_text(rng))
        n_tasks = 4 if rng.random() < 0.7 else None
        a, b = _outcome(beio.read_trace, path, n_tasks), _outcome(ref_read, path, n_tasks)
        assert a == b, open(path).read()
        n_err += a[0] == "err"
    assert 100 < n_err < 550  # both outcomes well represented


def _records(rng, n):
    out = []
    t = 0.0
    rates = rng.choice([0.25, 2.0, 3.0, 48.0], size=n)
    for i in range(n):
        t += float(rng.exponential(40.0))
        out.append((i, t, int(rng.integers(0, 4)), int(rng.integers(0, 3)),
                    float(rng.choice([1.0, rng.uniform(0, 1), 0.0])), float(rng.exponential(30.0)),
                    float(rates[i])))
    return out


def test_writers_match_reference_bytes(tmp_path):
    from besteffort import cli as ref_cli
    from besteffort import evalkit as ref_ek
    from besteffort import workload as ref_wl
    from besteffort.config import parse_config
    spec = parse_config().reward_spec()
    rng = np.random.default_rng(7)
    for trial in range(6):
        n = int(rng.integers(0, 400))
        recs = _records(rng, n)
        ours = EvalRun([RequestRecord(*r) for r in recs], "p", 4, 0)
        theirs = ref_ek.EvalRun([ref_ek.RequestRecord(*r) for r in recs], "p", 4, 0)
        p1, p2 = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
        beio.write_metrics_csv(ours, p1)
        ref_ek.write_metrics_csv(theirs, p2)
        assert open(p1, "rb").read() == open(p2, "rb").read()
        assert [vars(r) for r in beio.read_metrics_csv(p1)] == [vars(r) for r in ref_ek.read_metrics_csv(p2)]
        tr = ref_wl.WorkloadTrace([ref_wl.ArrivalEvent(r[1], r[2]) for r in recs],
                                  [ref_wl.SegmentMark(0, 3.0)] + ([ref_wl.SegmentMark(n // 2, 0.1)] if n else []),
                                  seed=trial)
        beio.write_trace(tr, p1)
        ref_wl.write_trace(tr, p2)
        assert open(p1, "rb").read() == open(p2, "rb").read()
        if n:
            assert beio.summary_row(ours, spec) == pytest.approx(ref_cli._summary_rows(theirs, spec), nan_ok=True)
            beio.write_per_rate([ours, ours], spec, p1)
            ref_cli._write_per_rate([theirs, theirs], spec, p2)
            assert open(p1, "rb").read() == open(p2, "rb").read()


def test_beqn1_matches_reference(tmp_path):
    from besteffort import policy as ref_pol
    for seed in range(4):
        rng_a, rng_b = np.random.default_rng(seed), np.random.default_rng(seed)
        T, M, H = 1 + seed, 2 + seed % 3, 32 * (1 + seed)
        ours = specs.QNetwork.init_random(T, M, H, rng_a)
        theirs = ref_pol.QNetwork.init_random(T, M, H, rng_b)
        for a, b in zip(ours.params(), theirs.params()):
            assert np.array_equal(a, b)
        p1, p2 = str(tmp_path / "a.beqn"), str(tmp_path / "b.beqn")
        specs.save_checkpoint(ours, p1)
        ref_pol.save_checkpoint(theirs, p2)
        blob = open(p1, "rb").read()
        assert blob == open(p2, "rb").read()
        # corrupted variants: same accept / error message
        head_end = blob.index(b"\n", blob.index(b"\n") + 1) + 1
        variants = [blob[:-1], blob + b"\0", b"BEQN2" + blob[5:], blob.replace(b"\n", b"\n\n", 1),
                    blob[:head_end - 1] + b" 7\n" + blob[head_end:], b"BEQN1\n0 3 32\n",
                    b"BEQN1\nx y z\n", b"", b"BEQN1", blob[:head_end + 5]]
        for v in variants:
            with open(p1, "wb") as f:
                f.write(v)
            outs = []
            for fn, kw in ((specs.load_checkpoint, {}), (ref_pol.load_checkpoint, {})):
                try:
                    q = fn(p1, **kw)
                    outs.append(("ok", [x.tolist() for x in q.params()]))
                except Exception as e:  # noqa: BLE001
                    outs.append(("err", type(e).__name__, str(e)))
            assert outs[0] == outs[1], v[:40]
        with open(p1, "wb") as f:
            f.write(blob)
        for kw in (dict(n_tasks=T), dict(n_tiers=M + 1), dict(n_tasks=T + 1, n_tiers=M)):
            e1 = e2 = None
            try:
                specs.load_checkpoint(p1, **kw)
            except Exception as e:  # noqa: BLE001
                e1 = str(e)
            try:
                ref_pol.load_checkpoint(p1, **kw)
            except Exception as e:  # noqa: BLE001
                e2 = str(e)
            assert e1 == e2


def test_qnetwork_views_share_the_flat_buffer():
    net = specs.QNetwork.init_random(4, 3, 64, np.random.default_rng(1))
    net.b1 = np.arange(64.0)
    assert np.array_equal(net.flat[8 * 64:8 * 64 + 64], np.arange(64.0))
    c = net.copy()
    c.w2[0, 0] = 123.0
    assert net.w2[0, 0] != 123.0
    net.load_from(c)
    assert net.w2[0, 0] == 123.0
    with pytest.raises(ValueError):
        net.w1 = np.zeros((3, 3))
