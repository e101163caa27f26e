# ncu --set full of the training-loop kernels (env step, commit, learner) at config-3 shape
mkdir -p gpurun_out
tag=${1:-tp}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"env_step|commit_fused|learner_partial|learner_update" -s 2000 -c 4 \
    -o gpurun_out/prof_train_$tag -f python tools/probe_train.py 4096 600 device > /dev/null 2> gpurun_out/prof_train_$tag.err
