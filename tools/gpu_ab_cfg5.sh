# A/B of library variants on config 5 (unpredictable-1/-2, estimated rate, 65,536 envs)
mkdir -p gpurun_out
rm -f gpurun_out/ab5.txt
for v in "$@"; do
  BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$v.so timeout 900 python -c "
import sys, json; sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
import configs_bench as c
r = c.config5()
print('$v', json.dumps({k: round(v['env_steps_per_s'] / 1e9, 4) for k, v in r.items() if isinstance(v, dict)}))
" >> gpurun_out/ab5.txt 2>&1
done
