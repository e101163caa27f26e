# tensor-core router: parity tests, throughput probe, ncu --set full of the kernel
mkdir -p gpurun_out
tag=${1:-rt}
timeout 600 python -m pytest tests/test_route_tc_gpu.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python tools/probe_route.py > gpurun_out/${tag}_probe.json 2> gpurun_out/${tag}_probe.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_route_tc_$tag -f python tools/probe_route.py 4194304 2 > /dev/null 2> gpurun_out/prof_route_tc_$tag.err
