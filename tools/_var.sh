for v in base NOFENCE NOLB NOWR NOLB_NOWR; do
  if [ $v = base ]; then unset BE200_LIB; else export BE200_LIB=$PWD/paper_2401_07886_b200/csrc/build_var/lib_$v.so; fi
  echo "== $v"; python tools/probe_train.py 4096 3000 graph 2>&1 | cut -c1-90
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:env_step -s 600 -c 30 --csv --log-file gpurun_out/var_$v.csv python tools/probe_train.py 4096 1000 device > /dev/null 2>&1
done
