# A/B at config 2 with KG = 3 for each tools/var/<name>/libhgs.so
for v in "$@"; do
  HGS_LIB=tools/var/$v/libhgs.so timeout 300 python bench.py --kg 3 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/abk_$v.json 2> gpurun_out/abk_$v.err || tail -3 gpurun_out/abk_$v.err
  python -c "import json;d=json.load(open('gpurun_out/abk_$v.json'));print('$v', round(d['value'],2), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
