# NCCL path on one GPU: world-1 NCCL test, bench under torchrun (world 1, NCCL),
# and the dev shared-GPU world-2 gloo mode
timeout 300 python -m pytest tests/test_distributed_gpu.py -q -m gpu 2>&1 | tail -2
NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-ref-engine > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err
echo "rc=$?"; grep -c "NCCL INFO" gpurun_out/torchrun1.err; python -c "import json;d=json.loads(open('gpurun_out/torchrun1.json').read().splitlines()[-1]);print(d['value'],d['n_gpus'],d['best_cut'],d['e2e']['value'])"
GSB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --no-ref-engine --no-e2e > gpurun_out/share2.json 2> gpurun_out/share2.err
echo "rc=$?"; tail -c 400 gpurun_out/share2.json
