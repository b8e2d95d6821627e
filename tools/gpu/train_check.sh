timeout 900 python -m pytest tests/test_gpu_train.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/pc_c4.json 2> gpurun_out/pc_c4.err; tail -3 gpurun_out/pc_c4.err
python -c "import json;d=json.load(open('gpurun_out/pc_c4.json'));print('C4', round(d['value'],1), 'it/s', {k:round(v,3) for k,v in d['stages_ms'].items()}, d['stage_rooflines'])"
