cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_streaming.py -q -x 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --no-cpu --no-extras 2>&1 | tail -4
} > gpurun_out/stream.txt 2>&1
