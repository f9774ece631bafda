cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 200 python tools/time_fused.py 5 256 fused 4
H3_FUSED_IMPL=dfma timeout 200 python tools/time_fused.py 5 256 fused 4
timeout 200 python tools/time_fused.py 5 128 fused 8
} > gpurun_out/n5.txt 2>&1
