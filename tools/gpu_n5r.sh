cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 300 python tools/time_two_pass.py
timeout 300 python tools/time_fused.py 5 256 two_pass 2
} > gpurun_out/n5r.txt 2>&1
