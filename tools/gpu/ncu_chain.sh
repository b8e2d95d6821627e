ncu --set full --clock-control none --import-source on -k regex:"k_chain_rule|k_preprocess|k_depth_keys" -s 3 -c 3 \
  -o gpurun_out/prof_chain python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_chain.log 2>&1
tail -2 gpurun_out/prof_chain.log
