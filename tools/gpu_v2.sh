cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
for c in 0 7 8 6; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/v2.txt 2>&1
