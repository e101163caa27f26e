#!/bin/bash
# Run on the GPU box (gpurun): launch list + one --set full capture of each hot kernel.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/launches_bench.json 2> gpurun_out/launches_bench.err
ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o gpurun_out/prof_rollout -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > /dev/null 2> gpurun_out/prof_rollout.err
ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -s 1 -c 1 \
    -o gpurun_out/prof_reduce -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > /dev/null 2> gpurun_out/prof_reduce.err
ls -la gpurun_out
