# training-loop profiles (config 3: 4096 envs, batch 512): launch list (warm caches)
# and --set full of the fused env step + commit and the fused learner
tag=${1:-r2w}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 1500 -c 60 --csv \
  --log-file gpurun_out/train_launches_$tag.csv python tools/probe_train.py 4096 1000 device > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"env_step_commit|learner_partial" -s 1500 -c 2 \
    -o gpurun_out/prof_train_$tag -f python tools/probe_train.py 4096 1000 device > /dev/null 2> gpurun_out/prof_train_$tag.err
ls -la gpurun_out/*$tag*
