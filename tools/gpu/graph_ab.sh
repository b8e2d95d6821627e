for m in eager graph eager graph; do
  if [ $m = graph ]; then f=--graph; else f=; fi
  python bench.py $f --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/gab_$m.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/gab_$m.json"))
print("$m", round(d["value"],1), round(d["fwd_frames_per_s"],1), d["gpu_launches"])
PY
done
