"""Fixture generator: evaluation traces for the statistical policy-parity test.

Test infrastructure only.  Eight `unpredictable-1` traces (the paper's Table-3
workload) made by the UNMODIFIED reference generator
(`make_trace`, pkg/src/besteffort/evalkit.py:141-151 ->
gen_unpredictable_time_based, workload.py:144-171) with the CLI's trial seeds
(`component_seed(0, "gen:unpredictable-1:<k>")`, cli.py:177, config.py:98-101).
Output: tests/golden/policy_traces.npz (arrival [K][N] f64, task [K][N] u8,
segment marks as CSR).  Usage:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_policy_traces.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("BE_REF_SRC", "/root/reference/pkg/src"))

from besteffort.config import component_seed  # noqa: E402
from besteffort.evalkit import make_trace, scenario_suite  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
K = 8


def main():
    sc = scenario_suite("unpredictable-1")
    arr, tsk, offs, ss, sr = [], [], [0], [], []
    for k in range(K):
        tr = make_trace(sc, 4, component_seed(0, f"gen:unpredictable-1:{k}"))
        arr.append([e.time_ms for e in tr.events])
        tsk.append([e.task_id for e in tr.events])
        ss.extend(m.start_index for m in tr.segment_marks)
        sr.extend(m.rate for m in tr.segment_marks)
        offs.append(len(ss))
    np.savez_compressed(os.path.join(HERE, "policy_traces.npz"), arrival=np.array(arr, np.float64),
                        task=np.array(tsk, np.uint8), seg_offsets=np.array(offs, np.int64),
                        seg_start=np.array(ss, np.int64), seg_rate=np.array(sr, np.float64),
                        scenario=np.array("unpredictable-1"), numpy=np.array(np.__version__))
    print("wrote", K, "traces")


if __name__ == "__main__":
    main()
