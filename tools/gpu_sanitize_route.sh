# compute-sanitizer (memcheck with API-error reporting off, racecheck, synccheck)
# over the tensor-core router tests: partial tiles, ties (every state re-evaluated),
# and one (T, M, H) shape per hidden width class
mkdir -p gpurun_out
tag=${1:-sanr}
SEL='test_route_tc_gpu.py::test_partial_tiles
test_route_tc_gpu.py::test_exact_ties_fall_back_and_take_the_first_maximum
test_route_tc_gpu.py::test_shapes'
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/${tag}_${tool}.log
  : > $out
  extra=""; [ $tool = memcheck ] && extra="--report-api-errors no"
  for t in $SEL; do
    echo "== $t" >> $out
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 \
      python -m pytest "tests/$t" -x -q -p no:cacheprovider >> $out 2>&1
    echo "exit $?" >> $out
  done
done
