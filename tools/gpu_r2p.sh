timeout 600 python -m pytest -q tests/test_errors_gpu.py > gpurun_out/r2p_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2p_pytest.log
tail -15 gpurun_out/r2p_pytest.log
bash tools/gpu_sanitize_r2.sh san2
