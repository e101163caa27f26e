"""Byte-identical CSV I/O (paper_2401_07886_b200.io) vs files written by the
reference's own writers (sha256 in tests/golden/csv_hashes.json, produced by
tests/golden/make_csv_golden.py): trace files (workload.py:258-267), metrics
(evalkit.py:300-305), summary (cli.py:145-195) and per-rate (cli.py:203-216)
CSVs; plus the validating trace reader's errors (workload.py:270-321)."""
import hashlib
import json
import os

import numpy as np
import pytest

import goldens
from paper_2401_07886_b200 import io as beio
from paper_2401_07886_b200.evalkit import EvalRun, RequestRecord
from paper_2401_07886_b200.specs import ArrivalEvent, SegmentMark, WorkloadTrace
from helpers import reward_of

HASHES = json.load(open(os.path.join(goldens.GOLDEN, "csv_hashes.json")))["runs"]


def sha(path):
    b = open(path, "rb").read()
    return [hashlib.sha256(b).hexdigest(), len(b)]


def eval_run(g):
    n = len(g["arrival"])
    rates = np.empty(n)
    starts = list(g["seg_start"]) + [n]
    for k in range(len(g["seg_start"])):
        rates[starts[k]:starts[k + 1]] = g["seg_rate"][k]
    recs = [RequestRecord(i, float(g["arrival"][i]), int(g["task"][i]), int(g["tier"][i]),
                          float(g["reward"][i]), float(g["realized"][i]), float(rates[i]))
            for i in range(n)]
    return EvalRun(records=recs, policy_id="golden", gpu_count=4, seed=0)


@pytest.mark.parametrize("name", sorted(HASHES))
def test_csv_bytes_match_reference(tmp_path, name):
    g = goldens.load(name)
    tr = WorkloadTrace([ArrivalEvent(float(t), int(k)) for t, k in zip(g["arrival"], g["task"])],
                       [SegmentMark(int(s), float(r)) for s, r in zip(g["seg_start"], g["seg_rate"])],
                       seed=12345)
    run = eval_run(g)
    spec = reward_of(g["meta"])
    p = {k: str(tmp_path / f"{k}.csv") for k in ("trace", "metrics", "summary", "per_rate")}
    beio.write_trace(tr, p["trace"])
    beio.write_metrics_csv(run, p["metrics"])
    beio.write_summary([run, run], spec, p["summary"])
    beio.write_per_rate([run, run], spec, p["per_rate"])
    for k in p:
        assert sha(p[k]) == HASHES[name][k], k
    back = beio.read_trace(p["trace"], n_tasks=4)
    assert back.events == tr.events and back.segment_marks == tr.segment_marks and back.seed == 12345
    recs = beio.read_metrics_csv(p["metrics"])
    assert [(r.tier_id, r.reward) for r in recs] == [(r.tier_id, r.reward) for r in run.records]


def test_read_trace_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    cases = ["# rng,pcg64\narrival_ms,task_id\n1.0,0\n0.5,1\n",   # not sorted
             "arrival_ms,task_id\n1.0\n",                         # 1 column
             "time,task\n1.0,0\n",                                # header
             "# segment,x,1.0\narrival_ms,task_id\n",             # malformed comment
             "arrival_ms,task_id\n1.0,7\n"]                       # unknown task
    for text in cases:
        bad.write_text(text)
        with pytest.raises(beio.TraceParseError) as ei:
            beio.read_trace(str(bad), n_tasks=4)
        assert str(bad) in str(ei.value)
    bad.write_text("# seed,3\n")
    with pytest.raises(beio.TraceParseError):
        beio.read_trace(str(bad))
