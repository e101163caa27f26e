mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rollout_gpu.py -x -q -k "random_configs" > gpurun_out/rc_pytest.log 2>&1; echo "exit $?" >> gpurun_out/rc_pytest.log
