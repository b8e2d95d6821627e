# Source-level capture of the fused surgery + Adam kernel at config 4
ncu --set full --clock-control none --import-source on -k regex:k_optim -s 1 -c 1 \
  -o /tmp/prof_optim python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_optim.log 2>&1
ncu -i /tmp/prof_optim.ncu-rep --page source --csv --print-source sass > gpurun_out/src_k_optim.csv 2>&1
ncu -i /tmp/prof_optim.ncu-rep --page raw --csv > gpurun_out/raw_k_optim.csv 2>&1
ls -la gpurun_out/src_k_optim.csv
