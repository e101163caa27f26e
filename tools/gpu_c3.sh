mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_learner_gpu.py tests/test_peer_exchange_gpu.py -x -q > gpurun_out/c3_pytest.log 2>&1; echo "exit $?" >> gpurun_out/c3_pytest.log
timeout 600 python tools/probe_train_var.py 3000 > gpurun_out/c3var.log 2>&1
