#!/bin/bash
# Router A/B: parity tests on the default library, then probe_route.py
# (4M states) for each library variant given as arguments, two passes.
# usage: gpurun -- bash tools/gpu_route_ab.sh TAG base v1 v2 ...
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_route_tc_gpu.py tests/test_policy_parity.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
for i in 1 2; do
  for v in "$@"; do
    L=$PWD/paper_2401_07886_b200/libbe200_$v.so; [ $v = cur ] && L=$PWD/paper_2401_07886_b200/libbe200.so
    echo -n "$v " >> gpurun_out/${tag}_probe.txt
    BE200_LIB=$L timeout 300 python tools/probe_route.py 4194304 50 >> gpurun_out/${tag}_probe.txt 2>>gpurun_out/${tag}_probe.err
  done
done
