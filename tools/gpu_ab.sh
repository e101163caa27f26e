# A/B: bench (no CPU leg) for each library variant given as arguments
mkdir -p gpurun_out
for v in "$@"; do
  BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-training > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', d['value'], d['kernel_ms'])" >> gpurun_out/ab.txt
done
