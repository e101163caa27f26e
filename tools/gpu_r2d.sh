# round-2: new/changed GPU tests, reducer prefetch A/B, config-3 policy record (pending 1<<16)
tag=${1:-r2d}
timeout 900 python -m pytest -q -x tests/test_step_gpu.py tests/test_reduce_gpu.py tests/test_training_dropin_gpu.py tests/test_replay_gpu.py tests/test_rollout_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
rm -f gpurun_out/${tag}_reduce.txt
for r in 1 2; do for v in red0_4 red4_4 red8_4 red8_8 red16_8; do
  BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$v.so timeout 300 python tools/probe_reduce.py >> gpurun_out/${tag}_reduce.txt 2>&1
done; done
timeout 1500 python tools/train_config3_policies.py --no-save > gpurun_out/${tag}_c3.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_reduce.txt; tail -3 gpurun_out/${tag}_c3.log
