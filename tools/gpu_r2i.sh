# round-2: rollout A/B (head vs constant-bank encode scales vs + evict-first trace loads)
rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh head c0 c1 head c0 c1
cat gpurun_out/ab.txt
