# Round profile set (exports CSV on the box; gpurun_out/ must stay < 64 MiB):
#  1. launch list of the default bench command (per-launch gpu__time_duration)
#  2. ncu --set full, one launch of every product kernel at config 2 -> raw CSV
#  3. ncu --set full of the training-step kernels at config 4 -> raw CSV
#  4. ncu --set full + source of the two compositors (kept as .ncu-rep)
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_c2.log 2>&1
ncu --set full --clock-control none \
  -k regex:"k_depth_keys|k_sort_plan|k_onesweep|k_rank_scatter|k_preprocess|k_tile_counts|k_scan_counts|k_duplicate|k_tile_ranges|k_composite|k_fixup|k_chain_rule" \
  -s 60 -c 60 -o /tmp/prof_c2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_c2.log 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv
ncu --set full --clock-control none -k regex:"k_loss|k_optim|k_composite_bwd|k_chain" -s 6 -c 6 \
  -o /tmp/prof_c4 python bench.py --config 4 --steps 1 --warmup 2 > gpurun_out/prof_c4.log 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > gpurun_out/prof_c4_raw.csv
ncu --set full --clock-control none --import-source on -k regex:"k_composite_fwd|k_composite_bwd" -s 4 -c 2 \
  -o gpurun_out/prof_comp python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_comp.log 2>&1
du -sh gpurun_out; ls -la gpurun_out
