ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd -s 2 -c 1 \
  -o gpurun_out/prof_bwd python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_bwd.log 2>&1
tail -2 gpurun_out/prof_bwd.log
