# round-2: fused tensor-core decision in the training env step — tests + throughput
tag=${1:-r2j}
timeout 900 python -m pytest -q -x tests/test_router_tc_step_gpu.py tests/test_learner_gpu.py tests/test_rollout_gpu.py tests/test_rollout_scale_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
rm -f gpurun_out/${tag}_train.txt
for E in 4096 65536; do for r in fp64 tc fp64 tc; do
  timeout 300 python tools/probe_train.py $E 2000 graph 1 $r >> gpurun_out/${tag}_train.txt 2>&1
done; done
tail -5 gpurun_out/${tag}_pytest.log; cut -c1-120 gpurun_out/${tag}_train.txt
