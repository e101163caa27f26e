# ncu --set full of the rollout kernel at bench shape (+ per-line attribution input)
tag=${1:-p}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o gpurun_out/prof_rollout_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training \
    > /dev/null 2> gpurun_out/prof_rollout_$tag.err
