# round-2: commit driven by the step's completion range — training tests + throughput
tag=${1:-r2m}
timeout 1200 python -m pytest -q -x tests/test_learner_gpu.py tests/test_replay_gpu.py tests/test_router_tc_step_gpu.py tests/test_training_dropin_gpu.py tests/test_peer_exchange_gpu.py tests/test_multirank_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
rm -f gpurun_out/${tag}_train.txt
for r in fp64 tc fp64 tc; do
  timeout 300 python tools/probe_train.py 4096 3000 graph 1 $r >> gpurun_out/${tag}_train.txt 2>&1
done
timeout 300 python tools/probe_train.py 65536 1000 graph 1 fp64 >> gpurun_out/${tag}_train.txt 2>&1
tail -3 gpurun_out/${tag}_pytest.log; cut -c1-110 gpurun_out/${tag}_train.txt
