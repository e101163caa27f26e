# compute-sanitizer over tools/sanitize_r2.py (round-2 kernels)
mkdir -p gpurun_out
tag=${1:-san2}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_r2.py > gpurun_out/${tag}_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_${tool}.log
  tail -4 gpurun_out/${tag}_${tool}.log
done
