# Source-level (SASS) instruction counts of both compositors, exported on the box.
set -x
for k in k_composite_fwd k_composite_bwd; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o /tmp/prof_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_$k.log 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>&1
  ls -la gpurun_out/src_$k.csv
done
