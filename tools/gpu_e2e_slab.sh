# multi-rank HostStepper (slab streaming) tests + bench e2e at N=1 and N=2 (gloo, one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_streaming.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --no-cpu --cells 256 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --cells 128 --no-extras --no-cpu 2>&1 | tail -3
} > gpurun_out/e2e_slab.txt 2>&1
