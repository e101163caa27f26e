timeout 900 python -m pytest -q -x tests/test_streaming_gpu.py tests/test_bench_gpu.py > gpurun_out/r2y_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2y_pytest.log; tail -3 gpurun_out/r2y_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-training --no-cpu-baseline > gpurun_out/r2y_bench.json 2> gpurun_out/r2y_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2y_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['value']/d['value'], d['reducer_roofline']['frac'])"
