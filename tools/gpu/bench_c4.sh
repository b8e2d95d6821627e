timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -5 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
