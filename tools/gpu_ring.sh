mkdir -p gpurun_out
for c in 64 256 1024; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --ring-capacity $c > gpurun_out/ring_$c.json 2> gpurun_out/ring_$c.err
  python -c "import json; d=json.load(open('gpurun_out/ring_$c.json')); print($c, d['value'], d['kernel_ms'])" >> gpurun_out/ring.txt 2>&1 || tail -2 gpurun_out/ring_$c.err >> gpurun_out/ring.txt
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:rollout_kernel -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ring-capacity 64 > gpurun_out/ring_ncu64.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:rollout_kernel -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ring_ncu_auto.txt 2>&1
