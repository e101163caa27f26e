# round-2: rollout A/B (old vs new encode division / task check), rollout tests
tag=${1:-r2e}
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh rold rnew rold rnew
timeout 900 python -m pytest -q -x tests/test_rollout_gpu.py tests/test_rollout_scale_gpu.py tests/test_known_answers_gpu.py > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
cat gpurun_out/ab.txt; tail -2 gpurun_out/${tag}_pytest.log
