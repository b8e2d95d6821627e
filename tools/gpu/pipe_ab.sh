# A/B of the multi-view pipeline at config 5 (64 views, 1M, 1080p):
# HGS_VIEW_PIPELINE 0 = sequential, 1 = forwards / backwards on two streams,
# 2 = + each view's chain rule on a third stream (two scratches)
timeout 900 python -m pytest tests/test_gpu_multiview.py -x -q 2>&1 | tail -2
for r in 1 2; do for v in 0 1 2; do
  HGS_VIEW_PIPELINE=$v timeout 600 python bench.py --config 5 --steps 3 --warmup 1 > gpurun_out/pipe_$v.json 2> gpurun_out/pipe_$v.err || tail -3 gpurun_out/pipe_$v.err
  python -c "import json;d=json.load(open('gpurun_out/pipe_$v.json'));print('pipeline $v', round(d['value'],1), d['unit'], round(d.get('ms_per_step'),2))"
done; done
HGS_VIEW_PIPELINE=2 HGS_PIPE_PRIO=bwd timeout 600 python bench.py --config 5 --steps 3 --warmup 1 > gpurun_out/pipe_2b.json 2> gpurun_out/pipe_2b.err
python -c "import json;d=json.load(open('gpurun_out/pipe_2b.json'));print('pipeline 2 prio bwd', round(d['value'],1))"
