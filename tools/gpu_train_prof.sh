mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv \
  --log-file gpurun_out/train_launches.csv python tools/probe_train.py 4096 60 host > /dev/null 2>&1
timeout 600 python -m pytest tests/test_learner_gpu.py -x -q > gpurun_out/tq_pytest.log 2>&1; echo "exit $?" >> gpurun_out/tq_pytest.log
