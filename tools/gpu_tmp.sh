rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh cur m96 t224 cur m96 t224
cat gpurun_out/ab.txt
