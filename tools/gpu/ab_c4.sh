# A/B at config 4 (KG = 3) for each tools/var/<name>/libhgs.so
for v in "$@"; do
  HGS_LIB=tools/var/$v/libhgs.so timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/ab4_$v.json 2> gpurun_out/ab4_$v.err || tail -3 gpurun_out/ab4_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab4_$v.json'));print('$v', round(d['value'],2), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
