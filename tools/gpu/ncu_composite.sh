# ncu --set full of the two compositors (one launch each) on the config-2 bench workload
set -x
ncu --set full --clock-control none --import-source on -k regex:k_composite -s 4 -c 2 \
  -o gpurun_out/prof_comp python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_comp.log 2>&1
tail -3 gpurun_out/prof_comp.log
ls -la gpurun_out
