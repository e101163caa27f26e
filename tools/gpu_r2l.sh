# round-2: fused tensor-core training step v2 (deferred image wait, double-buffered epilogue)
tag=${1:-r2l}
timeout 900 python -m pytest -q -x tests/test_router_tc_step_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
rm -f gpurun_out/${tag}_train.txt
for r in fp64 tc fp64 tc; do
  timeout 300 python tools/probe_train.py 4096 3000 graph 1 $r >> gpurun_out/${tag}_train.txt 2>&1
done
tail -3 gpurun_out/${tag}_pytest.log; cut -c1-110 gpurun_out/${tag}_train.txt
