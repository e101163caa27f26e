# round-2: rollout A/B (c1 vs lean) + ncu of the fused tensor-core training step
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh c1 lean c1 lean
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"env_step|prep_kernel" -s 400 -c 4 \
    -o gpurun_out/prof_steptc_r2k -f python tools/probe_train.py 4096 300 device 1 tc > /dev/null 2> gpurun_out/prof_steptc_r2k.err
cat gpurun_out/ab.txt
