rm -f gpurun_out/ab.txt
bash tools/gpu_ab.sh na ef2 na ef2
cat gpurun_out/ab.txt
for v in ef2; do
BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:rollout_kernel -s 1 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-training 2>/dev/null | grep -E "dram__" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
