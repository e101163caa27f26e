mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multirank_gpu.py -x -q > gpurun_out/multi_pytest.log 2>&1; echo "exit $?" >> gpurun_out/multi_pytest.log
