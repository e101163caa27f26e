# A/B of library variants on the training probe (config 3 shape)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/abt.txt
  BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$v.so timeout 600 python tools/probe_train.py 4096 5000 device >> gpurun_out/abt.txt 2>&1
done
