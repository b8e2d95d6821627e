ncu --set full --clock-control none -k regex:"k_loss|k_optim" -s 3 -c 3 \
  -o gpurun_out/prof_train python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/prof_train.log 2>&1
tail -2 gpurun_out/prof_train.log
