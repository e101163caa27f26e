mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "exit $?" >> gpurun_out/t_pytest.log
timeout 300 python tools/probe_train.py 1 3000 > gpurun_out/t_probe_e1.log 2>&1
timeout 3000 python tools/train_gpu_policies.py 7 8 9 10 > gpurun_out/t_policies.log 2>&1
mkdir -p gpurun_out/policies && cp tests/golden/gpu_trained_seed*.beqn gpurun_out/policies/
