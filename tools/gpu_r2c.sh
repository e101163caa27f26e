# round-2: full GPU suite, smoke, headline bench (driver invocation), config-3 policy parity record
tag=${1:-r2c}
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-training > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 1200 python tools/train_config3_policies.py --no-save > gpurun_out/${tag}_c3.log 2>&1
tail -15 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_smoke.log; tail -3 gpurun_out/${tag}_c3.log
