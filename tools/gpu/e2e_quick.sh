python tools/e2e_ab.py 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/be.json 2> gpurun_out/be.err; grep "e2e step" gpurun_out/be.err
python -c "import json;d=json.load(open('gpurun_out/be.json'));print(d['value'], d['e2e']['value'])"
