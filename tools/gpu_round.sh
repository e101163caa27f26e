# round-2 checkpoint: full GPU suite, smoke, the driver's bench invocation (both arms),
# ncu launch list + --set full of the rollout (current code)
tag=${1:-r2n}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${tag}_smi.txt 2>&1; nproc > gpurun_out/${tag}_nproc.txt
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-training \
    > gpurun_out/launches_bench_${tag}.json 2> gpurun_out/launches_bench_${tag}.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o gpurun_out/prof_rollout_${tag} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training \
    > /dev/null 2> gpurun_out/prof_rollout_${tag}.err
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_smoke.log | tail -2; tail -2 gpurun_out/${tag}_bench.err
