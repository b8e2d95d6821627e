# A/B of the front end's stream layout: "name:aux_priority" per run, the
# library tools/var/<name>/libhgs.so, HGS_AUX_PRIORITY=<aux_priority>
for spec in "$@"; do
  v=${spec%%:*}; p=${spec#*:}
  HGS_AUX_PRIORITY=$p HGS_LIB=tools/var/$v/libhgs.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/abf_$v$p.json 2> gpurun_out/abf_$v$p.err || tail -3 gpurun_out/abf_$v$p.err
  python -c "import json;d=json.load(open('gpurun_out/abf_$v$p.json'));print('$v prio $p', round(d['value'],1), 'fwd', round(d['fwd_frames_per_s'],1), {k:round(x,3) for k,x in d['stages_ms'].items()})"
done
