# A/B: headline bench stage times for each tools/var/<name>/libhgs.so
for v in "$@"; do
  HGS_LIB=tools/var/$v/libhgs.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err || tail -3 gpurun_out/ab_$v.err
  python -c "import json,sys;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['value'],1), 'it/s fwd', round(d['fwd_frames_per_s'],1), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
