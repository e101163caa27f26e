"""Fixture generator: sha256 of the CSV files the UNMODIFIED reference writes.

Test infrastructure only (criterion-12-style file-hash
parity).  For golden runs (tests/golden/run_*.npz, produced by the reference's
run_eval) it rebuilds the reference WorkloadTrace / EvalRun and writes, with the
reference's own writers,
  write_trace        (workload.py:258-267)
  write_metrics_csv  (evalkit.py:300-305)
  summary CSV        (cli.py:184-195 via _summary_rows, cli.py:145-160)
  per-rate CSV       (cli.py:203-216, stable scenarios)
and records each file's sha256 and size in tests/golden/csv_hashes.json.
Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_csv_golden.py
"""
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from besteffort import cli  # noqa: E402
from besteffort.evalkit import write_metrics_csv  # noqa: E402
from besteffort.workload import ArrivalEvent, SegmentMark, WorkloadTrace, write_trace  # noqa: E402
from make_evalstats_golden import eval_run, load, spec_of  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = ["stable_trained", "unpredictable-1_trained", "hellaswag-copa-soft_mixed1", "quantized_static2"]


def sha(path):
    b = open(path, "rb").read()
    return hashlib.sha256(b).hexdigest(), len(b)


def main():
    out = {}
    d = tempfile.mkdtemp()
    for name in RUNS:
        g = load(name)
        tr = WorkloadTrace([ArrivalEvent(float(t), int(k)) for t, k in zip(g["arrival"], g["task"])],
                           [SegmentMark(int(s), float(r)) for s, r in zip(g["seg_start"], g["seg_rate"])],
                           seed=12345)
        run = eval_run(g)
        spec = spec_of(g["meta"])
        files = {"trace": os.path.join(d, "t.csv"), "metrics": os.path.join(d, "m.csv"),
                 "summary": os.path.join(d, "s.csv"), "per_rate": os.path.join(d, "p.csv")}
        write_trace(tr, files["trace"])
        write_metrics_csv(run, files["metrics"])
        rows = [cli._summary_rows(run, spec), cli._summary_rows(run, spec)]
        keys = list(rows[0].keys())
        with open(files["summary"], "w", encoding="utf-8", newline="\n") as f:  # cli.py:184-195
            f.write("trial," + ",".join(keys) + "\n")
            for k, row in enumerate(rows):
                f.write(f"{k}," + ",".join(repr(row[key]) if isinstance(row[key], float)
                                           else str(row[key]) for key in keys) + "\n")
        cli._write_per_rate([run, run], spec, files["per_rate"])
        out[name] = {k: sha(p) for k, p in files.items()}
    json.dump(dict(runs=out, numpy=np.__version__), open(os.path.join(HERE, "csv_hashes.json"), "w"),
              indent=1)
    print(json.dumps(out, indent=1)[:400])


if __name__ == "__main__":
    main()
