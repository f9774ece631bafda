cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA_CFG=20 timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
for c in 0 20 21 11 0 20; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/lean.txt 2>&1
