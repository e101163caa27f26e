bash tools/gpu_train_quick.sh t3
bash tools/gpu_train_prof_full.sh t3
