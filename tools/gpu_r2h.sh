# round-2: tensor-core router on the training env step — tests + throughput at E = 4096 / 16384 / 65536
tag=${1:-r2h}
timeout 900 python -m pytest -q -x tests/test_router_tc_step_gpu.py tests/test_step_gpu.py tests/test_learner_gpu.py tests/test_route_tc_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
rm -f gpurun_out/${tag}_train.txt
for E in 4096 16384 65536; do for r in fp64 tc; do
  timeout 300 python tools/probe_train.py $E 2000 graph 1 $r >> gpurun_out/${tag}_train.txt 2>&1
done; done
tail -5 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_train.txt
