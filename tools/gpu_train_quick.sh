# quick GPU iteration on the training path: learner/step/multirank parity tests,
# the config-3 probe (device + graph modes) and a torch.profiler kernel table (warm caches)
mkdir -p gpurun_out
tag=${1:-t}
timeout 900 python -m pytest tests/test_learner_gpu.py tests/test_step_gpu.py tests/test_multirank_gpu.py tests/test_rollout_gpu.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python tools/probe_train.py 4096 3000 device > gpurun_out/${tag}_train.log 2>&1
timeout 300 python tools/probe_train.py 4096 3000 graph >> gpurun_out/${tag}_train.log 2>&1
timeout 300 python tools/prof_train.py 4096 > gpurun_out/${tag}_prof.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-training > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
