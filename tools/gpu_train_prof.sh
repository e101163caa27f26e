mkdir -p gpurun_out
lib=${1:-}
[ -n "$lib" ] && export BE200_LIB=$PWD/paper_2401_07886_b200/libbe200_$lib.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 70 --csv \
  --log-file gpurun_out/train_launches.csv python tools/probe_train.py 4096 1000 device > /dev/null 2>&1
