# bench.py at N=1 (full) and N=2 (two ranks on one GPU via gloo, with the DP training probe)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b1.json 2> gpurun_out/b1.err
BE_DIST_BACKEND=gloo OMP_NUM_THREADS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --steps 2 --warmup 3 --envs 4096 --requests 2000 \
  --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
echo "exit $?" >> gpurun_out/b2.err
