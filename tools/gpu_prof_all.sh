# round-2 profiles: ncu launch list of the bench command, --set full of the rollout,
# reducer, tensor-core router and the training-loop kernels (step, commit, learner)
tag=${1:-r2a}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-training \
    > gpurun_out/launches_bench_$tag.json 2> gpurun_out/launches_bench_$tag.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o gpurun_out/prof_rollout_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training \
    > /dev/null 2> gpurun_out/prof_rollout_$tag.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -s 1 -c 1 \
    -o gpurun_out/prof_reduce_$tag -f python tools/probe_reduce.py > /dev/null 2> gpurun_out/prof_reduce_$tag.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_route_tc_$tag -f python tools/probe_route.py 4194304 2 > /dev/null 2> gpurun_out/prof_route_tc_$tag.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"env_step|commit_fused|learner_partial|learner_update|prep_kernel" -s 2000 -c 5 \
    -o gpurun_out/prof_train_$tag -f python tools/probe_train.py 4096 600 device > /dev/null 2> gpurun_out/prof_train_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 70 --csv \
  --log-file gpurun_out/train_launches_$tag.csv python tools/probe_train.py 4096 1000 device > /dev/null 2>&1
ls -la gpurun_out/*$tag*
