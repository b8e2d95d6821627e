# parity + headline bench + config 4 (quick perf iteration)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pc_c2.json 2> gpurun_out/pc_c2.err; tail -3 gpurun_out/pc_c2.err
python -c "import json;d=json.load(open('gpurun_out/pc_c2.json'));print('C2', round(d['value'],1), 'it/s fwd', round(d['fwd_frames_per_s'],1), {k:round(v,3) for k,v in d['stages_ms'].items()})"
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/pc_c4.json 2> gpurun_out/pc_c4.err; tail -3 gpurun_out/pc_c4.err
python -c "import json;d=json.load(open('gpurun_out/pc_c4.json'));print('C4', round(d['value'],1), 'it/s', {k:round(v,3) for k,v in d['stages_ms'].items()})"
