#!/bin/bash
# One gpurun call: GPU parity tests, the bench line (both arms), the ncu launch
# list and one --set full capture of each hot kernel.  Outputs in gpurun_out/.
# usage: gpurun --timeout 3000 -- bash tools/gpu_round.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_$tag.txt 2>&1
nproc > gpurun_out/nproc_$tag.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
timeout 300 python tools/probe_train.py 4096 3000 device > gpurun_out/train_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-training \
    > gpurun_out/launches_bench_$tag.json 2> gpurun_out/launches_bench_$tag.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o gpurun_out/prof_rollout_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training \
    > /dev/null 2> gpurun_out/prof_rollout_$tag.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -s 1 -c 1 \
    -o gpurun_out/prof_reduce_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training \
    > /dev/null 2> gpurun_out/prof_reduce_$tag.err
timeout 300 python tools/probe_route.py > gpurun_out/route_$tag.json 2> gpurun_out/route_$tag.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_route_tc_$tag -f python tools/probe_route.py 4194304 2 > /dev/null 2> gpurun_out/prof_route_tc_$tag.err
ls -la gpurun_out
timeout 1200 python tools/configs_bench.py > gpurun_out/configs_$tag.log 2>&1 && cp gpurun_out/configs.json gpurun_out/configs_$tag.json
