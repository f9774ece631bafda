cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 200 python tools/time_fused.py 3 128 fused 20
timeout 200 python tools/time_fused.py 3 128 two_pass 10
timeout 200 python tools/time_fused.py 3 256 fused 10
timeout 200 python tools/time_fused.py 3 512 fused 6
timeout 200 python tools/time_fused.py 5 256 fused 4
} > gpurun_out/z.txt 2>&1
