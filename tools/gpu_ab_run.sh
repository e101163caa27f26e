mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rollout_gpu.py -x -q > gpurun_out/s2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/s2_pytest.log
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh b2 b3
