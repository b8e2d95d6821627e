# Full bench lines for the round record: default (config 2, with e2e + CPU
# baseline), reference arm, config 3, 4, 5, KG=3 at config 2, fast mode.
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -2 gpurun_out/b_c2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 600 python bench.py --config 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 600 python bench.py --config 4 --steps 20 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 1 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 600 python bench.py --kg 3 --no-e2e --no-cpu-baseline > gpurun_out/b_c2kg3.json 2> gpurun_out/b_c2kg3.err
timeout 600 python bench.py --fast --no-e2e --no-cpu-baseline > gpurun_out/b_c2fast.json 2> gpurun_out/b_c2fast.err
for f in gpurun_out/b_*.json; do echo $f; cut -c1-400 $f; done
