cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 200 python tools/time_fused.py 5 256 fused 4
timeout 300 python tools/time_fused.py 5 256 two_pass 2
timeout 300 python tools/time_two_pass.py 2>&1 | tail -1
} > gpurun_out/n5p.txt 2>&1
