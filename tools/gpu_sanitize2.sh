# memcheck re-run of the tests whose first launch reported a driver API error:
# eager module loading, and memory checking with API-error reporting off
mkdir -p gpurun_out
tag=${1:-san2}
out=gpurun_out/${tag}_memcheck.log
: > $out
for t in "test_reduce_gpu.py::test_selection_and_secondary_reducers_match_reference" \
         "test_tracegen_gpu.py::test_scenarios_generate" "test_route_tc_gpu.py::test_partial_tiles[129]"; do
  echo "== EAGER $t" >> $out
  CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 5 \
      python -m pytest "tests/$t" -x -q -p no:cacheprovider >> $out 2>&1
  echo "exit $?" >> $out
  echo "== no-api-errors $t" >> $out
  timeout 900 compute-sanitizer --tool memcheck --report-api-errors no --error-exitcode 9 --print-limit 5 \
      python -m pytest "tests/$t" -x -q -p no:cacheprovider >> $out 2>&1
  echo "exit $?" >> $out
done
