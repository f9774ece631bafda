cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA_CFG=22 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "separable or degenerate or slab or instab" 2>&1 | tail -2
for c in 0 22 23 24 0 22; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/2cta.txt 2>&1
