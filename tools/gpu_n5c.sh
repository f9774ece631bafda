cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA5_CFG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "separable or degenerate" 2>&1 | tail -1
for c in 0 1 2; do H3_DMMA5_CFG=$c timeout 200 python tools/time_fused.py 5 256 fused 4; done
} > gpurun_out/n5c.txt 2>&1
