# A/B the library variants given as arguments (bench without CPU leg / training)
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh "$@"
