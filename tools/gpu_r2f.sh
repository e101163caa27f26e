# round-2: rollout A/B (old vs exact-mul variant), new drop-in tests
tag=${1:-r2f}
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh rold rnew rold rnew
timeout 1200 python -m pytest -q tests/test_reference_objects_gpu.py tests/test_cli_backend_gpu.py tests/test_step_gpu.py tests/test_training_dropin_gpu.py tests/test_rollout_gpu.py tests/test_lib_symbols.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
cat gpurun_out/ab.txt; tail -15 gpurun_out/${tag}_pytest.log
