# Multi-rank logic check on a 1-GPU box: 2 ranks share cuda:0 over gloo.
export HGS_DIST_BACKEND=gloo CUDA_VISIBLE_DEVICES=0
for cfg in "--steps 3 --warmup 3 --no-e2e" "--config 4 --steps 2 --warmup 3" "--config 5 --steps 1 --warmup 1"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 $cfg > gpurun_out/mr.json 2> gpurun_out/mr.err; echo "rc=$? $cfg"; tail -2 gpurun_out/mr.err | cut -c1-300; cut -c1-300 gpurun_out/mr.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --impl reference --steps 1 --warmup 0 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/mr_ref.json
