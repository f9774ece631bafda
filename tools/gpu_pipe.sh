cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA_CFG=27 timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
for c in 0 26 27 28 0 26 27; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/pipe.txt 2>&1
