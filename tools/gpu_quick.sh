# quick GPU iteration: rollout parity tests + a short bench line (no CPU baseline / training probe)
mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests/test_rollout_gpu.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-training > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
