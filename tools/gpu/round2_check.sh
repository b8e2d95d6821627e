# GPU suite + multi-rank logic check (2 gloo ranks on one GPU) + default bench
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -12
export HGS_DIST_BACKEND=gloo
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/mr2.json 2> gpurun_out/mr2.err; echo "rc=$?"; tail -3 gpurun_out/mr2.err | cut -c1-300; cut -c1-400 gpurun_out/mr2.json
timeout 900 python bench.py --gpus 2 --config 5 --steps 1 --warmup 1 > gpurun_out/mr5.json 2> gpurun_out/mr5.err; echo "rc=$?"; tail -3 gpurun_out/mr5.err | cut -c1-300; cut -c1-400 gpurun_out/mr5.json
unset HGS_DIST_BACKEND
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/c5.json 2> gpurun_out/c5.err; cut -c1-300 gpurun_out/c5.json
timeout 600 python bench.py --steps 20 > gpurun_out/c2.json 2> gpurun_out/c2.err; tail -2 gpurun_out/c2.err; cut -c1-2500 gpurun_out/c2.json
