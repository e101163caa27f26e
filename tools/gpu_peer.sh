mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_peer_exchange_gpu.py -x -q > gpurun_out/peer_pytest.log 2>&1; echo "exit $?" >> gpurun_out/peer_pytest.log
