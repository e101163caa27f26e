mkdir -p gpurun_out
tag=${1:-cf}
timeout 900 python -m pytest tests/test_rollout_gpu.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-training > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 1200 python tools/configs_bench.py > gpurun_out/${tag}_configs.log 2>&1 && cp gpurun_out/configs.json gpurun_out/configs_${tag}.json
