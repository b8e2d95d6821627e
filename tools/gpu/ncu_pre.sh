# Source-level capture of the preprocess at config 2
ncu --set full --clock-control none --import-source on -k regex:k_preprocess -s 2 -c 1 \
  -o /tmp/prof_pre python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_pre.log 2>&1
ncu -i /tmp/prof_pre.ncu-rep --page source --csv --print-source sass > gpurun_out/src_k_preprocess.csv 2>&1
ncu -i /tmp/prof_pre.ncu-rep --page details --csv > gpurun_out/det_k_preprocess.csv 2>&1
ls -la gpurun_out/src_k_preprocess.csv
