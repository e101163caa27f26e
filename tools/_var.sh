for v in base PREPWL CW2 CW8 base; do
  if [ $v = base ]; then unset BE200_LIB; else export BE200_LIB=$PWD/paper_2401_07886_b200/csrc/build_var/lib_$v.so; fi
  echo "== $v"; python tools/probe_train.py 4096 3000 graph 2>&1 | cut -c1-90
done
